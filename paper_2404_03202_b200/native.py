"""ctypes binding of the product library ``libosplat_b200.so`` (include/osplat.h).

This module is the Python-side mirror of the reference interface for the hot path:

* ``render(cloud, pose, W, H)``         -> proj/include/omnisplat/rasterizer.hpp:85-86
* ``Context.backward(frame, d_image)``  -> proj/include/omnisplat/gradients.hpp:43-44
* ``Context.adam_step(cfg, extent, it)``-> proj/include/omnisplat/trainer.hpp:80-81
* ``osplat_render`` / ``osplat_cloud_*`` reference C ABI (proj/include/omnisplat/capi.h)

There is no fallback: if the shared library is missing the import fails, and every call that
reaches a CUDA error raises :class:`OsplatError`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .scenes import Cloud

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSPLAT_LIB", os.path.join(HERE, "libosplat_b200.so"))  # override: A/B builds

OK, INVALID_ARGUMENT, IO, PARSE, VALIDATION, UNSUPPORTED, RUNTIME = range(7)
STATUS_NAMES = {0: "OK", 1: "INVALID_ARGUMENT", 2: "IO", 3: "PARSE", 4: "VALIDATION", 5: "UNSUPPORTED",
                6: "RUNTIME"}


class OsplatError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"osplat status {STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_u32p = C.POINTER(C.c_uint32)
_lp = C.POINTER(C.c_long)
_vp = C.c_void_p


class FrameView(C.Structure):
    _fields_ = [("rgb", _vp), ("transmittance", _vp), ("contributors", _vp), ("last_contrib", _vp),
                ("width", C.c_int), ("height", C.c_int)]


class GpuView(C.Structure):
    _fields_ = [("params", _vp), ("grads", _vp), ("adam_m", _vp), ("adam_v", _vp), ("d_screen", _vp),
                ("screen_norm_sum", _vp), ("screen_hits", _vp), ("n", C.c_size_t), ("stride", C.c_size_t),
                ("planes", C.c_int), ("sh_degree", C.c_int), ("active_sh_degree", C.c_int),
                ("adam_step", C.c_long), ("max_radius_px", _vp)]


class EditSummary(C.Structure):
    _fields_ = [("cloned", C.c_long), ("split", C.c_long), ("pruned", C.c_long), ("final_count", C.c_size_t)]


PROGRESS_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_long, C.c_double, C.c_size_t)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (make -C paper_2404_03202_b200)")
    lib = C.CDLL(LIB_PATH)
    S = C.c_int  # osplat_status
    sig = {
        "osplat_version": (C.c_char_p, []),
        "osplat_last_error": (C.c_char_p, []),
        "osplat_set_threads": (None, [C.c_int]),
        "osplat_cloud_load": (S, [C.c_char_p, C.POINTER(_vp)]),
        "osplat_cloud_save": (S, [_vp, C.c_char_p]),
        "osplat_cloud_count": (C.c_size_t, [_vp]),
        "osplat_cloud_free": (None, [_vp]),
        "osplat_config_create": (S, [C.POINTER(_vp)]),
        "osplat_config_set": (S, [_vp, C.c_char_p, C.c_char_p]),
        "osplat_config_free": (None, [_vp]),
        "osplat_render": (S, [_vp, _dp, C.c_int, C.c_int, C.POINTER(_vp)]),
        "osplat_image_width": (C.c_int, [_vp]),
        "osplat_image_height": (C.c_int, [_vp]),
        "osplat_image_pixels": (_dp, [_vp]),
        "osplat_image_free": (None, [_vp]),
        "osplat_cloud_create": (S, [C.c_size_t, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, C.POINTER(_vp)]),
        "osplat_cloud_read": (S, [_vp, _dp, _dp, _dp, _dp, _dp, _ip, _ip]),
        "osplat_gpu_create": (S, [C.c_int, _vp, _vp, C.POINTER(_vp)]),
        "osplat_gpu_free": (None, [_vp]),
        "osplat_gpu_count": (C.c_size_t, [_vp]),
        "osplat_gpu_set_active_sh_degree": (S, [_vp, C.c_int]),
        "osplat_gpu_set_deterministic": (S, [_vp, C.c_int]),
        "osplat_gpu_set_strict_guard": (S, [_vp, C.c_int]),
        "osplat_nccl_unique_id": (S, [C.POINTER(C.c_ubyte)]),
        "osplat_gpu_dp_init": (S, [_vp, C.c_int, C.c_int, C.POINTER(C.c_ubyte)]),
        "osplat_gpu_dp_step": (S, [_vp, _vp, C.c_double, C.c_long]),
        "osplat_gpu_download": (S, [_vp, C.POINTER(_vp)]),
        "osplat_gpu_synchronize": (S, [_vp]),
        "osplat_gpu_render": (S, [_vp, _dp, C.c_int, C.c_int, _dp, C.POINTER(_vp)]),
        "osplat_frame_free": (None, [_vp]),
        "osplat_frame_width": (C.c_int, [_vp]),
        "osplat_frame_height": (C.c_int, [_vp]),
        "osplat_frame_image": (S, [_vp, _dp]),
        "osplat_frame_pixels": (S, [_vp, _fp, _fp, _ip, _ip]),
        "osplat_frame_projections": (S, [_vp, _u8p, _dp, _dp, _dp, _fp, _i32p, _u32p]),
        "osplat_frame_tiles": (S, [_vp, _ip, _ip, C.POINTER(C.c_size_t), _u32p, _u32p]),
        "osplat_frame_device": (S, [_vp, C.POINTER(FrameView)]),
        "osplat_gpu_view_buffers": (S, [_vp, C.POINTER(GpuView)]),
        "osplat_gpu_backward": (S, [_vp, _vp, _dp, C.c_int]),
        "osplat_gpu_backward_device": (S, [_vp, _vp, _vp, C.c_int]),
        "osplat_gpu_gradients": (S, [_vp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _lp]),
        "osplat_gpu_zero_grad": (S, [_vp]),
        "osplat_gpu_reset_screen_stats": (S, [_vp]),
        "osplat_gpu_adam_step": (S, [_vp, _vp, C.c_double, C.c_long, C.c_int]),
        "osplat_gpu_adam_step_range": (S, [_vp, _vp, C.c_double, C.c_long, C.c_int, C.c_size_t, C.c_size_t]),
        "osplat_gpu_l1_loss": (S, [_vp, _vp, _vp, C.c_double, C.POINTER(_vp), _dp]),
        "osplat_gpu_loss": (S, [_vp, _vp, _vp, C.c_double, C.c_double, C.POINTER(_vp), _dp]),
        "osplat_gpu_train_view": (S, [_vp, _dp, C.c_int, C.c_int, _vp, C.c_int, C.c_double, C.c_double, _dp]),
        "osplat_gpu_launch_count": (C.c_longlong, []),
        "osplat_gpu_profile": (S, [_vp, C.c_int, C.c_int]),
        "osplat_gpu_profile_read": (S, [_vp, _dp, _lp, C.c_int]),
        "osplat_kernel_name": (C.c_char_p, [C.c_int]),
        "osplat_gpu_observe": (S, [_vp, _vp]),
        "osplat_gpu_densify_and_prune": (S, [_vp, _vp, C.c_double, C.c_ulonglong, C.c_int, C.POINTER(EditSummary)]),
        "osplat_gpu_reset_opacity": (S, [_vp, C.c_double]),
        "osplat_gpu_max_radius": (S, [_vp, _dp]),
        "osplat_mix64": (C.c_ulonglong, [C.c_ulonglong]),
        "osplat_gpu_save_state": (S, [_vp, C.c_char_p, C.c_long]),
        "osplat_gpu_load_state": (S, [_vp, C.c_char_p, _lp]),
        "osplat_image_create": (S, [C.c_int, C.c_int, _dp, C.POINTER(_vp)]),
        "osplat_metrics": (S, [_vp, _vp, _dp, _dp]),
        "osplat_gpu_eval": (S, [_vp, C.c_size_t, _dp, C.POINTER(_vp), _u8p, C.c_char_p, C.c_int, C.POINTER(_vp)]),
        "osplat_report_view_count": (C.c_size_t, [_vp]),
        "osplat_report_view": (S, [_vp, C.c_size_t, _ip, _dp, _dp]),
        "osplat_report_mean": (S, [_vp, _dp, _dp, _dp, _dp]),
        "osplat_report_mode": (C.c_char_p, [_vp]),
        "osplat_report_free": (None, [_vp]),
        "osplat_gpu_train": (S, [_vp, _vp, C.c_size_t, _dp, C.POINTER(_vp), _u8p, C.c_double, C.c_long, C.c_char_p,
                                 PROGRESS_FN, C.c_void_p]),
        "osplat_frame_work": (S, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
        "osplat_frame_splats": (S, [_vp, C.POINTER(C.c_size_t), _i32p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]),
        "osplat_gpu_upload": (S, [_vp, _vp]),
        "osplat_gpu_train_view_async": (S, [_vp, _dp, C.c_int, C.c_int, _vp, C.c_int, C.c_double, C.c_double,
                                            C.c_void_p]),
        "osplat_loss_value": (C.c_double, [_dp, C.c_double, C.c_int, C.c_int, C.c_double]),
        "osplat_gpu_render_projected": (S, [_vp, C.c_size_t, _i32p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int,
                                            C.c_int, _dp, _u32p, _i32p, C.POINTER(_vp)]),
    }
    ab_build = "OSPLAT_LIB" in os.environ  # A/B runs may load older builds without newer entry points
    for name, (res, args) in sig.items():
        if ab_build and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
# osplat_frame_splats / osplat_gpu_render_projected per-record arrays, in argument order
SPLAT_FIELDS = ("gaussian_id", "p", "cov", "conic", "radius", "depth", "color", "alpha_base", "t")
KERNEL_COUNT = 11  # OSPLAT_KERNEL_COUNT
EXPORTED = ("osplat_version osplat_last_error osplat_set_threads osplat_cloud_load osplat_cloud_save "
            "osplat_cloud_count osplat_cloud_free osplat_config_create osplat_config_set osplat_config_free "
            "osplat_render osplat_image_width osplat_image_height osplat_image_pixels osplat_image_free").split()


def check(status: int):
    if status != OK:
        raise OsplatError(status, lib.osplat_last_error().decode())


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def loss_value(sums, lambda_ssim: float, width: int, height: int, mask: float = 0.0) -> float:
    """osplat_loss_value: the loss from osplat_gpu_train_view_async's sums."""
    a = np.ascontiguousarray(sums, dtype=np.float64)
    return float(lib.osplat_loss_value(_p(a), lambda_ssim, width, height, mask))


def nccl_unique_id() -> bytes:
    """osplat_nccl_unique_id: 128 bytes to hand to every rank's Context.dp_init."""
    buf = (C.c_ubyte * 128)()
    check(lib.osplat_nccl_unique_id(buf))
    return bytes(buf)


def version() -> str:
    return lib.osplat_version().decode()


def launch_count() -> int:
    return int(lib.osplat_gpu_launch_count())


def transform_of(pose12: np.ndarray) -> np.ndarray:
    """12-double pose (R row-major, t) -> row-major 4x4 world->camera (capi.cpp:88-95)."""
    t = np.eye(4)
    t[:3, :3] = np.asarray(pose12[:9], dtype=np.float64).reshape(3, 3)
    t[:3, 3] = pose12[9:12]
    return np.ascontiguousarray(t)


# --------------------------------------------------------------------------- host handles

class HostCloud:
    """Owning wrapper of an ``osplat_cloud`` handle (reference GaussianCloud on the host)."""

    def __init__(self, handle):
        self.handle = handle

    @staticmethod
    def from_cloud(cloud: Cloud) -> "HostCloud":
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (cloud.positions, cloud.sh, cloud.rotations, cloud.log_scales, cloud.opacity_logits)]
        h = _vp()
        check(lib.osplat_cloud_create(cloud.n, cloud.sh_degree, cloud.active_sh_degree,
                                      *[_p(a) for a in arrs], C.byref(h)))
        return HostCloud(h)

    @staticmethod
    def load(path: str) -> "HostCloud":
        h = _vp()
        check(lib.osplat_cloud_load(path.encode(), C.byref(h)))
        return HostCloud(h)

    def save(self, path: str):
        check(lib.osplat_cloud_save(self.handle, path.encode()))

    def __len__(self):
        return int(lib.osplat_cloud_count(self.handle))

    def to_cloud(self) -> Cloud:
        deg, act = C.c_int(0), C.c_int(0)
        check(lib.osplat_cloud_read(self.handle, None, None, None, None, None, C.byref(deg), C.byref(act)))
        n = len(self)
        bc = (deg.value + 1) ** 2
        pos, sh, rot = np.zeros((n, 3)), np.zeros((n, bc, 3)), np.zeros((n, 4))
        ls, op = np.zeros((n, 3)), np.zeros(n)
        check(lib.osplat_cloud_read(self.handle, _p(pos), _p(sh), _p(rot), _p(ls), _p(op), None, None))
        return Cloud(pos, sh, rot, ls, op, deg.value, act.value)

    def __del__(self):
        if getattr(self, "handle", None):
            lib.osplat_cloud_free(self.handle)
            self.handle = None


def osplat_render(cloud: HostCloud, pose12, width: int, height: int, out: np.ndarray | None = None) -> np.ndarray:
    """The reference drop-in entry point (capi.h:73-74): host cloud in, H x W x 3 double out
    (copied into `out` when given, e.g. a viewer's reused frame buffer)."""
    with osplat_image(cloud, pose12, width, height) as px:
        if out is None:
            return px.copy()
        np.copyto(out, px)
        return out


def osplat_metrics(a: np.ndarray, b: np.ndarray) -> tuple[float, float]:
    """The reference osplat_metrics (capi.h:90-92): (PSNR dB capped at 99, SSIM) of two H x W x 3
    images, computed on the GPU through osplat_image handles."""
    hs = []
    try:
        for im in (a, b):
            im = np.ascontiguousarray(im, dtype=np.float64)
            if im.ndim != 3 or im.shape[2] != 3:
                raise ValueError("osplat_metrics: images must be H x W x 3")
            h = _vp()
            check(lib.osplat_image_create(im.shape[1], im.shape[0], _p(im), C.byref(h)))
            hs.append(h)
        ps, ss = C.c_double(0.0), C.c_double(0.0)
        check(lib.osplat_metrics(hs[0], hs[1], C.byref(ps), C.byref(ss)))
        return ps.value, ss.value
    finally:
        for h in hs:
            lib.osplat_image_free(h)


class osplat_image:
    """Context manager over an osplat_render result: a zero-copy numpy view of the osplat_image's
    pixels, valid until the block exits (osplat_image_free)."""

    def __init__(self, cloud: HostCloud, pose12, width: int, height: int):
        self.cloud, self.t, self.size = cloud, transform_of(pose12), (width, height)
        self.img = _vp()

    def __enter__(self) -> np.ndarray:
        check(lib.osplat_render(self.cloud.handle, _p(self.t), self.size[0], self.size[1], C.byref(self.img)))
        w, h = lib.osplat_image_width(self.img), lib.osplat_image_height(self.img)
        return np.ctypeslib.as_array(lib.osplat_image_pixels(self.img), shape=(h, w, 3))

    def __exit__(self, *exc):
        lib.osplat_image_free(self.img)
        self.img = _vp()


class Config:
    """``osplat_config`` (TrainConfig) with string setters (dataio.cpp:570-605)."""

    def __init__(self, **fields):
        self.handle = _vp()
        check(lib.osplat_config_create(C.byref(self.handle)))
        for k, v in fields.items():
            self.set(k, v)

    def set(self, key: str, value):
        check(lib.osplat_config_set(self.handle, key.encode(), str(value).encode()))

    def __del__(self):
        if getattr(self, "handle", None):
            lib.osplat_config_free(self.handle)
            self.handle = None


# --------------------------------------------------------------------------- device context

class Frame:
    """Retained forward state of one render (the reference RenderOutput)."""

    def __init__(self, ctx: "Context", handle):
        self.ctx = ctx
        self.handle = handle
        self.width = lib.osplat_frame_width(handle)
        self.height = lib.osplat_frame_height(handle)

    def image(self) -> np.ndarray:
        out = np.zeros((self.height, self.width, 3))
        check(lib.osplat_frame_image(self.handle, _p(out)))
        return out

    def pixels(self):
        H, W = self.height, self.width
        rgb = np.zeros((H, W, 3), dtype=np.float32)
        T = np.zeros((H, W), dtype=np.float32)
        con = np.zeros((H, W), dtype=np.int32)
        last = np.zeros((H, W), dtype=np.int32)
        check(lib.osplat_frame_pixels(self.handle, _p(rgb, _fp), _p(T, _fp), _p(con, _ip), _p(last, _ip)))
        return rgb, T, con, last

    def projections(self):
        n = self.ctx.n
        vis = np.zeros(n, dtype=np.uint8)
        p, conic, op = np.zeros((n, 2)), np.zeros((n, 3)), np.zeros(n)
        col = np.zeros((n, 3), dtype=np.float32)
        rect = np.zeros((n, 4), dtype=np.int32)
        touched = np.zeros(n, dtype=np.uint32)
        check(lib.osplat_frame_projections(self.handle, _p(vis, _u8p), _p(p), _p(conic), _p(op), _p(col, _fp),
                                           _p(rect, _i32p), _p(touched, _u32p)))
        return dict(visible=vis.astype(bool), p=p, conic=conic, opacity=op, color=col, rect=rect,
                    touched=touched)

    def tiles(self):
        tx, ty, m = C.c_int(0), C.c_int(0), C.c_size_t(0)
        check(lib.osplat_frame_tiles(self.handle, C.byref(tx), C.byref(ty), C.byref(m), None, None))
        ranges = np.zeros((tx.value * ty.value, 2), dtype=np.uint32)
        ids = np.zeros(max(m.value, 1), dtype=np.uint32)
        check(lib.osplat_frame_tiles(self.handle, None, None, None, _p(ranges, _u32p), _p(ids, _u32p)))
        return tx.value, ty.value, ranges, ids[:m.value]

    def splats(self) -> dict:
        """Full SplatProjection records (osplat_frame_splats): visible Gaussians in ascending id for a
        render, the given records for a render_projected frame."""
        n = C.c_size_t(0)
        check(lib.osplat_frame_splats(self.handle, C.byref(n), *([None] * 9)))
        k = n.value
        out = dict(gaussian_id=np.zeros(k, dtype=np.int32), p=np.zeros((k, 2)), cov=np.zeros((k, 3)),
                   conic=np.zeros((k, 3)), radius=np.zeros(k), depth=np.zeros(k), color=np.zeros((k, 3)),
                   alpha_base=np.zeros(k), t=np.zeros((k, 3)))
        ptrs = [_p(out["gaussian_id"], _i32p)] + [_p(out[f]) for f in SPLAT_FIELDS[1:]]
        check(lib.osplat_frame_splats(self.handle, C.byref(n), *ptrs))
        return out

    def work(self):
        """(forward pairs visited, backward pairs, tile instances) — needs count_work profiling."""
        f, b, m = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
        check(lib.osplat_frame_work(self.handle, C.byref(f), C.byref(b), C.byref(m)))
        return f.value, b.value, m.value

    def device(self) -> FrameView:
        v = FrameView()
        check(lib.osplat_frame_device(self.handle, C.byref(v)))
        return v

    def free(self):
        if self.handle:
            lib.osplat_frame_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()


class Context:
    """``osplat_gpu``: device-resident parameters, gradients and Adam state on one GPU."""

    def __init__(self, cloud: Cloud | HostCloud, device: int = 0, stream: int | None = None):
        hc = cloud if isinstance(cloud, HostCloud) else HostCloud.from_cloud(cloud)
        self.handle = _vp()
        # stream: None -> the library creates its own stream; an int is a cudaStream_t handle, where
        # 0 (torch's default stream) means the legacy default stream (cudaStreamLegacy = 0x1).
        if stream is None:
            s = None
        else:
            s = C.c_void_p(stream if stream != 0 else 0x1)
        check(lib.osplat_gpu_create(device, s, hc.handle, C.byref(self.handle)))
        self.device = device
        v = self.view()
        self.n, self.stride, self.planes, self.sh_degree = v.n, v.stride, v.planes, v.sh_degree
        self.basis_count = (v.sh_degree + 1) ** 2

    def view(self) -> GpuView:
        v = GpuView()
        check(lib.osplat_gpu_view_buffers(self.handle, C.byref(v)))
        return v

    def eval(self, poses, images, is_test=None, split: str = "test", perspective_crop: bool = False) -> dict:
        """osplat_gpu_eval (osplat_eval / run_eval over in-memory views): per-view PSNR / SSIM, means,
        seconds per frame and FPS (render only, steady clock), mode."""
        T = np.ascontiguousarray(np.stack([transform_of(p) for p in poses]), dtype=np.float64)
        handles = []
        try:
            for im in images:
                im = np.ascontiguousarray(im, dtype=np.float64)
                h = _vp()
                check(lib.osplat_image_create(im.shape[1], im.shape[0], _p(im), C.byref(h)))
                handles.append(h)
            arr = (_vp * len(handles))(*handles)
            flags = None if is_test is None else np.ascontiguousarray(is_test, dtype=np.uint8)
            rep = _vp()
            check(lib.osplat_gpu_eval(self.handle, len(handles), _p(T), arr,
                                      _p(flags, _u8p) if flags is not None else None, split.encode(),
                                      int(perspective_crop), C.byref(rep)))
        finally:
            for h in handles:
                lib.osplat_image_free(h)
        try:
            views = []
            for i in range(lib.osplat_report_view_count(rep)):
                fi, ps, ss = C.c_int(0), C.c_double(0), C.c_double(0)
                check(lib.osplat_report_view(rep, i, C.byref(fi), C.byref(ps), C.byref(ss)))
                views.append((fi.value, ps.value, ss.value))
            mp, ms, spf, fps = C.c_double(0), C.c_double(0), C.c_double(0), C.c_double(0)
            check(lib.osplat_report_mean(rep, C.byref(mp), C.byref(ms), C.byref(spf), C.byref(fps)))
            return {"views": views, "mean_psnr": mp.value, "mean_ssim": ms.value, "seconds_per_frame": spf.value,
                    "fps": fps.value, "mode": lib.osplat_report_mode(rep).decode()}
        finally:
            lib.osplat_report_free(rep)

    def dp_init(self, world: int, rank: int, unique_id: bytes):
        """osplat_gpu_dp_init: this context becomes rank `rank` of a `world`-GPU data-parallel job
        (NCCL communicator owned by the library)."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        check(lib.osplat_gpu_dp_init(self.handle, world, rank, buf))

    def dp_step(self, config: "Config | None", extent: float, iteration: int):
        """osplat_gpu_dp_step: reduce-scatter of the gradients, Adam on this rank's shard,
        all-gather of the parameters (NCCL, on the context stream)."""
        check(lib.osplat_gpu_dp_step(self.handle, config.handle if config else None, extent, iteration))

    def set_strict_guard(self, on: bool = True):
        """Strict (provable) T-stop guard band in K3 instead of the default 2^-10 band."""
        check(lib.osplat_gpu_set_strict_guard(self.handle, int(bool(on))))

    def set_deterministic(self, on: bool = True):
        """Deterministic backward (fixed-order reduction, bit-identical gradients run to run)."""
        check(lib.osplat_gpu_set_deterministic(self.handle, int(bool(on))))

    def set_active_sh_degree(self, d: int):
        check(lib.osplat_gpu_set_active_sh_degree(self.handle, d))

    def render(self, pose12, width: int, height: int, background=(0.0, 0.0, 0.0)) -> Frame:
        t = transform_of(pose12)
        bg = np.ascontiguousarray(background, dtype=np.float64)
        h = _vp()
        check(lib.osplat_gpu_render(self.handle, _p(t), width, height, _p(bg), C.byref(h)))
        return Frame(self, h)

    def upload(self, cloud: Cloud | HostCloud):
        """Replace the device cloud (osplat_gpu_upload)."""
        hc = cloud if isinstance(cloud, HostCloud) else HostCloud.from_cloud(cloud)
        check(lib.osplat_gpu_upload(self.handle, hc.handle))
        self._refresh()

    def render_projected(self, splats: dict, width: int, height: int, background=(0.0, 0.0, 0.0),
                         grid=None) -> Frame:
        """bin_to_tiles + blend_forward over host SplatProjection records (a dict with the keys of
        Frame.splats(); 't' is ignored). grid: None (bin on the device) or (ranges [tiles, 2],
        entries [M]) as Frame.tiles() returns them for such a frame."""
        k = len(splats["depth"])
        ids = np.ascontiguousarray(splats.get("gaussian_id", np.arange(k)), dtype=np.int32)
        arrs = [np.ascontiguousarray(splats[f], dtype=np.float64) for f in SPLAT_FIELDS[1:8]]
        bg = np.ascontiguousarray(background, dtype=np.float64)
        offs = ents = None
        if grid is not None:
            ranges, entries = grid
            ranges = np.asarray(ranges, dtype=np.int64)
            offs = np.ascontiguousarray(np.concatenate([[0], np.cumsum(ranges[:, 1] - ranges[:, 0])]), dtype=np.uint32)
            ents = np.ascontiguousarray(np.concatenate([entries[a:b] for a, b in ranges] + [np.zeros(0)]),
                                        dtype=np.int32)
        h = _vp()
        check(lib.osplat_gpu_render_projected(self.handle, k, _p(ids, _i32p), *[_p(a) for a in arrs], width, height,
                                              _p(bg), None if offs is None else _p(offs, _u32p),
                                              None if ents is None else _p(ents, _i32p), C.byref(h)))
        return Frame(self, h)

    def backward(self, frame: Frame, d_image: np.ndarray, accumulate: bool = False):
        d = np.ascontiguousarray(d_image, dtype=np.float64)
        assert d.shape == (frame.height, frame.width, 3)
        check(lib.osplat_gpu_backward(self.handle, frame.handle, _p(d), int(accumulate)))

    def backward_device(self, frame: Frame, d_image_ptr: int, accumulate: bool = False):
        check(lib.osplat_gpu_backward_device(self.handle, frame.handle, C.c_void_p(d_image_ptr), int(accumulate)))

    def gradients(self):
        n, bc = self.n, self.basis_count
        out = dict(d_position=np.zeros((n, 3)), d_sh=np.zeros((n, bc, 3)), d_rotation=np.zeros((n, 4)),
                   d_log_scale=np.zeros((n, 3)), d_opacity_logit=np.zeros(n), d_screen=np.zeros((n, 2)),
                   screen_norm_sum=np.zeros(n), screen_hits=np.zeros(n, dtype=np.int64))
        check(lib.osplat_gpu_gradients(self.handle, *[_p(out[k]) for k in (
            "d_position", "d_sh", "d_rotation", "d_log_scale", "d_opacity_logit", "d_screen",
            "screen_norm_sum")], _p(out["screen_hits"], _lp)))
        return out

    def zero_grad(self):
        check(lib.osplat_gpu_zero_grad(self.handle))

    def reset_screen_stats(self):
        check(lib.osplat_gpu_reset_screen_stats(self.handle))

    def adam_step(self, config: Config | None, extent: float, iteration: int, zero_grad: bool = False,
                  begin: int = 0, count: int | None = None):
        """adam_step (trainer.cpp:143-178); with begin/count only that flat element range (a shard)."""
        if begin == 0 and count is None:
            check(lib.osplat_gpu_adam_step(self.handle, config.handle if config else None, extent, iteration,
                                           int(zero_grad)))
        else:
            check(lib.osplat_gpu_adam_step_range(self.handle, config.handle if config else None, extent, iteration,
                                                 int(zero_grad), begin, count if count is not None else 2**63))

    def loss(self, frame: Frame, gt_ptr: int, lambda_ssim: float = 0.2, mask_bottom_fraction: float = 0.0,
             want_value=True):
        """loss() (trainer.cpp:25-71) against a device planar target; returns (value, d_image ptr)."""
        d = _vp()
        val = C.c_double(0.0)
        check(lib.osplat_gpu_loss(self.handle, frame.handle, C.c_void_p(gt_ptr), lambda_ssim, mask_bottom_fraction,
                                  C.byref(d), C.byref(val) if want_value else None))
        return val.value, d.value

    def l1_loss(self, frame: Frame, gt_ptr: int, mask_bottom_fraction: float = 0.0, want_value=True):
        return self.loss(frame, gt_ptr, 0.0, mask_bottom_fraction, want_value)

    def train_view(self, pose12, width: int, height: int, gt, gt_on_device: bool, lambda_ssim: float = 0.2,
                   mask: float = 0.0) -> float:
        """render -> loss -> backward(accumulate); gt is a host numpy array (3,H,W) float32 or a
        pointer (int) to host (gt_on_device False) or device memory."""
        t = transform_of(pose12)
        loss = C.c_double(0.0)
        ptr = C.c_void_p(gt) if isinstance(gt, int) else gt.ctypes.data_as(C.c_void_p)
        check(lib.osplat_gpu_train_view(self.handle, _p(t), width, height, ptr, int(gt_on_device), lambda_ssim, mask,
                                        C.byref(loss)))
        return loss.value

    def train_view_noloss(self, pose12, width: int, height: int, gt, gt_on_device: bool, lambda_ssim: float = 0.2,
                          mask: float = 0.0):
        """train_view without reading the loss back (no host synchronisation at the end)."""
        t = transform_of(pose12)
        ptr = C.c_void_p(gt) if isinstance(gt, int) else gt.ctypes.data_as(C.c_void_p)
        check(lib.osplat_gpu_train_view(self.handle, _p(t), width, height, ptr, int(gt_on_device), lambda_ssim, mask,
                                        None))

    def train_view_async(self, pose12, width: int, height: int, gt, gt_on_device: bool, sums_ptr: int | None,
                         lambda_ssim: float = 0.2, mask: float = 0.0):
        """osplat_gpu_train_view_async: the step is enqueued, nothing waited for; the 4 loss sums land
        at sums_ptr (pinned host memory) once the stream gets there (osplat_loss_value turns them
        into the loss after synchronize())."""
        t = transform_of(pose12)
        ptr = C.c_void_p(gt) if isinstance(gt, int) else gt.ctypes.data_as(C.c_void_p)
        check(lib.osplat_gpu_train_view_async(self.handle, _p(t), width, height, ptr, int(gt_on_device), lambda_ssim,
                                              mask, None if sums_ptr is None else C.c_void_p(sums_ptr)))

    def profile(self, timing: bool = True, count_work: bool = False):
        check(lib.osplat_gpu_profile(self.handle, int(timing), int(count_work)))

    def profile_read(self, reset: bool = True) -> dict:
        """{kernel family: (total ms, launches)} since the last reset (synchronizes)."""
        ms = np.zeros(KERNEL_COUNT)
        cnt = np.zeros(KERNEL_COUNT, dtype=np.int64)
        check(lib.osplat_gpu_profile_read(self.handle, _p(ms), _p(cnt, _lp), int(reset)))
        return {lib.osplat_kernel_name(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(KERNEL_COUNT)}

    # ---- densification control (trainer.cpp:180-280) and the training loop
    def observe(self, frame: Frame):
        check(lib.osplat_gpu_observe(self.handle, frame.handle))

    def densify_and_prune(self, config: Config | None, extent: float, rng_seed: int, radius_prune_active: bool) -> dict:
        e = EditSummary()
        check(lib.osplat_gpu_densify_and_prune(self.handle, config.handle if config else None, extent,
                                               C.c_ulonglong(rng_seed & 0xFFFFFFFFFFFFFFFF), int(radius_prune_active),
                                               C.byref(e)))
        self._refresh()
        return {"cloned": e.cloned, "split": e.split, "pruned": e.pruned, "final_count": e.final_count}

    def reset_opacity(self, ceiling: float):
        check(lib.osplat_gpu_reset_opacity(self.handle, ceiling))

    def max_radius(self) -> np.ndarray:
        out = np.zeros(self.view().n)
        check(lib.osplat_gpu_max_radius(self.handle, _p(out)))
        return out

    def save_state(self, path: str, iteration: int):
        check(lib.osplat_gpu_save_state(self.handle, path.encode(), iteration))

    def load_state(self, path: str) -> int:
        it = C.c_long(0)
        check(lib.osplat_gpu_load_state(self.handle, path.encode(), C.byref(it)))
        return it.value

    def train(self, config: Config | None, poses, images, is_test=None, extent: float = 0.0, start_iteration: int = 0,
              output_dir: str | None = None, progress=None):
        """osplat_gpu_train: Trainer::run over in-memory views (poses: list of pose12, images: list of
        H x W x 3 float64 arrays). progress(iteration, loss, gaussians) on log iterations."""
        views = len(poses)
        T = np.ascontiguousarray(np.stack([transform_of(p) for p in poses]), dtype=np.float64)
        handles = []
        for im in images:
            im = np.ascontiguousarray(im, dtype=np.float64)
            h = _vp()
            check(lib.osplat_image_create(im.shape[1], im.shape[0], _p(im), C.byref(h)))
            handles.append(h)
        arr = (_vp * views)(*handles)
        flags = None if is_test is None else np.ascontiguousarray(is_test, dtype=np.uint8)
        cb = PROGRESS_FN(lambda user, it, loss, n: progress(it, loss, n)) if progress else PROGRESS_FN()
        try:
            check(lib.osplat_gpu_train(self.handle, config.handle if config else None, views, _p(T), arr,
                                       _p(flags, _u8p) if flags is not None else None, extent, start_iteration,
                                       output_dir.encode() if output_dir else None, cb, None))
        finally:
            for h in handles:
                lib.osplat_image_free(h)
            self._refresh()

    def _refresh(self):
        v = self.view()
        self.n, self.stride, self.planes, self.sh_degree = v.n, v.stride, v.planes, v.sh_degree
        self.basis_count = (v.sh_degree + 1) ** 2

    def download(self) -> Cloud:
        h = _vp()
        check(lib.osplat_gpu_download(self.handle, C.byref(h)))
        return HostCloud(h).to_cloud()

    def synchronize(self):
        check(lib.osplat_gpu_synchronize(self.handle))

    def free(self):
        if getattr(self, "handle", None):
            lib.osplat_gpu_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()
