"""ctypes binding of the two oracle libraries — TEST INFRASTRUCTURE ONLY.

``load("port")``      -> oracle/build/liboracle.so   (our C restatement, oracle/oracle.c)
``load("reference")`` -> oracle/_ref/libref_oracle.so (the reference's own sources)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": os.path.join(HERE, "build", "liboracle.so"),
    "reference": os.path.join(HERE, "_ref", "libref_oracle.so"),
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


class _Cloud(C.Structure):
    _fields_ = [("n", C.c_int), ("sh_degree", C.c_int), ("active_sh_degree", C.c_int),
                ("positions", _dp), ("sh", _dp), ("rotations", _dp), ("log_scales", _dp),
                ("opacity_logits", _dp)]


class _Grads(C.Structure):
    _fields_ = [("d_position", _dp), ("d_sh", _dp), ("d_rotation", _dp), ("d_log_scale", _dp),
                ("d_opacity_logit", _dp), ("d_screen", _dp), ("screen_norm_sum", _dp),
                ("screen_hits", _lp)]


class _Adam(C.Structure):
    _fields_ = [("m_position", _dp), ("v_position", _dp), ("m_sh", _dp), ("v_sh", _dp),
                ("m_rotation", _dp), ("v_rotation", _dp), ("m_scale", _dp), ("v_scale", _dp),
                ("m_opacity", _dp), ("v_opacity", _dp), ("step", C.c_long)]


class _AdamCfg(C.Structure):
    _fields_ = [("iterations", C.c_long), ("lr_position_init", C.c_double),
                ("lr_position_final", C.c_double), ("lr_sh_dc", C.c_double),
                ("lr_sh_rest", C.c_double), ("lr_opacity", C.c_double), ("lr_scale", C.c_double),
                ("lr_rotation", C.c_double)]


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


@dataclass
class Grads:
    """GradientBuffer mirror (gradients.hpp:16-36), reference layouts."""
    d_position: np.ndarray
    d_sh: np.ndarray
    d_rotation: np.ndarray
    d_log_scale: np.ndarray
    d_opacity_logit: np.ndarray
    d_screen: np.ndarray
    screen_norm_sum: np.ndarray
    screen_hits: np.ndarray

    @staticmethod
    def zeros(n: int, bc: int) -> "Grads":
        return Grads(np.zeros((n, 3)), np.zeros((n, bc, 3)), np.zeros((n, 4)), np.zeros((n, 3)),
                     np.zeros(n), np.zeros((n, 2)), np.zeros(n), np.zeros(n, dtype=np.int64))


@dataclass
class AdamState:
    m_position: np.ndarray
    v_position: np.ndarray
    m_sh: np.ndarray
    v_sh: np.ndarray
    m_rotation: np.ndarray
    v_rotation: np.ndarray
    m_scale: np.ndarray
    v_scale: np.ndarray
    m_opacity: np.ndarray
    v_opacity: np.ndarray
    step: int = 0

    @staticmethod
    def zeros(n: int, bc: int) -> "AdamState":
        z = lambda *s: np.zeros(s)
        return AdamState(z(n, 3), z(n, 3), z(n, bc, 3), z(n, bc, 3), z(n, 4), z(n, 4), z(n, 3),
                         z(n, 3), z(n), z(n), 0)


@dataclass
class AdamConfig:
    """TrainConfig learning-rate fields with the reference defaults (trainer.hpp:19-51)."""
    iterations: int = 7000
    lr_position_init: float = 1.6e-4
    lr_position_final: float = 1.6e-6
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 2.5e-3 / 20.0
    lr_opacity: float = 5e-2
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3


@dataclass
class DensifyConfig:
    """TrainConfig densification fields with the reference defaults (trainer.hpp:19-51)."""
    densify_grad_threshold: float = 2e-4
    scale_split_threshold: float = 0.01
    split_factor: float = 1.6
    prune_opacity: float = 0.005
    prune_scale_world: float = 0.1
    prune_radius_px: float = 20.0


class _DensifyCfg(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("densify_grad_threshold", "scale_split_threshold", "split_factor",
                                          "prune_opacity", "prune_scale_world", "prune_radius_px")]


class _Edit(C.Structure):
    _fields_ = [("cloned", C.c_long), ("split", C.c_long), ("pruned", C.c_long), ("final_count", C.c_long)]


ADAM_FIELDS = ("m_position", "v_position", "m_sh", "v_sh", "m_rotation", "v_rotation", "m_scale", "v_scale",
               "m_opacity", "v_opacity")


@dataclass
class Frame:
    width: int
    height: int
    gaussian_id: np.ndarray
    p: np.ndarray
    cov: np.ndarray
    conic: np.ndarray
    radius: np.ndarray
    depth: np.ndarray
    color: np.ndarray
    alpha: np.ndarray
    t: np.ndarray
    tiles_x: int
    tiles_y: int
    offsets: np.ndarray
    items: np.ndarray
    rgb: np.ndarray
    T: np.ndarray
    contributors: np.ndarray
    last_contrib: np.ndarray
    handle: object = None

    def tile_gaussian_lists(self):
        """Per tile, the Gaussian ids in blend order."""
        ids = self.gaussian_id[self.items] if self.items.size else self.items
        return [ids[self.offsets[t]:self.offsets[t + 1]] for t in range(self.tiles_x * self.tiles_y)]


class Oracle:
    def __init__(self, kind: str = "port"):
        path = PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.kind = kind
        lib = C.CDLL(path)
        self.lib = lib
        lib.oracle_render.restype = C.c_void_p
        lib.oracle_render.argtypes = [C.POINTER(_Cloud), _dp, C.c_int, C.c_int, _dp]
        lib.oracle_reference_render.restype = C.c_void_p
        lib.oracle_reference_render.argtypes = [C.POINTER(_Cloud), _dp, C.c_int, C.c_int, _dp]
        lib.oracle_frame_free.argtypes = [C.c_void_p]
        lib.oracle_blend_projections.restype = C.c_void_p
        lib.oracle_blend_projections.argtypes = [C.c_int, _ip] + [_dp] * 7 + [C.c_int, C.c_int, _dp, _lp, _ip]
        lib.oracle_frame_num_projections.restype = C.c_int
        lib.oracle_frame_num_projections.argtypes = [C.c_void_p]
        lib.oracle_frame_projections.argtypes = [C.c_void_p, _ip] + [_dp] * 8
        lib.oracle_frame_tile_count.restype = C.c_long
        lib.oracle_frame_tile_count.argtypes = [C.c_void_p, _ip, _ip]
        lib.oracle_frame_tile_lists.argtypes = [C.c_void_p, _lp, _ip]
        lib.oracle_frame_pixels.argtypes = [C.c_void_p, _dp, _dp, _ip, _ip]
        lib.oracle_backward.restype = C.c_int
        lib.oracle_backward.argtypes = [C.c_void_p, _dp, C.POINTER(_Cloud), _dp, C.c_int, C.c_int,
                                        C.POINTER(_Grads)]
        lib.oracle_adam_step.argtypes = [C.POINTER(_Cloud), C.POINTER(_Grads), C.POINTER(_Adam),
                                         C.POINTER(_AdamCfg), C.c_double, C.c_long]
        lib.oracle_loss.restype = C.c_double
        lib.oracle_loss.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, _dp]
        lib.oracle_metrics.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, _dp]
        lib.oracle_densify_and_prune.restype = C.c_int
        lib.oracle_densify_and_prune.argtypes = [C.POINTER(_Cloud), _dp, _lp, _dp, C.POINTER(_Adam),
                                                 C.POINTER(_DensifyCfg), C.c_double, C.c_ulonglong, C.c_int,
                                                 C.POINTER(_Cloud), C.POINTER(_Adam), C.POINTER(_Edit)]
        lib.oracle_reset_opacity.argtypes = [C.POINTER(_Cloud), C.c_double]
        lib.oracle_mt64_draws.argtypes = [C.c_ulonglong, C.c_long, C.POINTER(C.c_ulonglong)]
        lib.oracle_mix64.restype = C.c_ulonglong
        lib.oracle_mix64.argtypes = [C.c_ulonglong]
        lib.oracle_set_threads.argtypes = [C.c_int]
        lib.oracle_threads.restype = C.c_int
        lib.oracle_kind.restype = C.c_char_p
        lib.oracle_last_seconds.restype = C.c_double

    # ------------------------------------------------------------------ helpers
    @staticmethod
    def _cloud(cloud, keep):
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (cloud.positions, cloud.sh, cloud.rotations, cloud.log_scales, cloud.opacity_logits)]
        keep.extend(arrs)
        return _Cloud(cloud.n, cloud.sh_degree, cloud.active_sh_degree, *[_ptr(a) for a in arrs])

    def set_threads(self, n: int):
        self.lib.oracle_set_threads(int(n))

    def threads(self) -> int:
        return int(self.lib.oracle_threads())

    def last_seconds(self) -> float:
        """Steady-clock time of the last render/backward/adam_step/loss call (no marshalling)."""
        return float(self.lib.oracle_last_seconds())

    # ------------------------------------------------------------------ API
    def render(self, cloud, pose, width, height, background=(0.0, 0.0, 0.0), brute_force=False,
               keep_handle=False) -> Frame:
        keep = []
        c = self._cloud(cloud, keep)
        pose = np.ascontiguousarray(pose, dtype=np.float64)
        bg = np.ascontiguousarray(background, dtype=np.float64)
        fn = self.lib.oracle_reference_render if brute_force else self.lib.oracle_render
        h = fn(C.byref(c), _ptr(pose), width, height, _ptr(bg))
        if not h:
            raise RuntimeError("oracle render failed")
        try:
            return self._frame(h, width, height, keep_handle)
        finally:
            if not keep_handle:
                self.lib.oracle_frame_free(h)

    def blend_projections(self, splats: dict, width, height, background=(0.0, 0.0, 0.0), grid=None) -> Frame:
        """bin_to_tiles + blend_forward over host SplatProjection records (rasterizer.cpp:57-157).
        splats: dict of per-record arrays (gaussian_id, p, cov, conic, radius, depth, color, alpha_base);
        grid: None, or (offsets [tiles+1], items [M]) = the TileGrid to blend."""
        n = len(splats["depth"])
        gid = np.ascontiguousarray(splats.get("gaussian_id", np.arange(n)), dtype=np.int32)
        arrs = [np.ascontiguousarray(splats[k], dtype=np.float64)
                for k in ("p", "cov", "conic", "radius", "depth", "color", "alpha_base")]
        bg = np.ascontiguousarray(background, dtype=np.float64)
        offs = items = None
        if grid is not None:
            offs = np.ascontiguousarray(grid[0], dtype=np.int64)
            items = np.ascontiguousarray(grid[1] if len(grid[1]) else np.zeros(1), dtype=np.int32)
        h = self.lib.oracle_blend_projections(n, _ptr(gid, _ip), *[_ptr(a) for a in arrs], width, height, _ptr(bg),
                                              None if offs is None else _ptr(offs, _lp),
                                              None if items is None else _ptr(items, _ip))
        if not h:
            raise RuntimeError("oracle blend_projections failed")
        try:
            return self._frame(h, width, height, False)
        finally:
            self.lib.oracle_frame_free(h)

    def _frame(self, h, W, H, keep_handle) -> Frame:
        lib = self.lib
        n = lib.oracle_frame_num_projections(h)
        gid = np.zeros(n, dtype=np.int32)
        p, cov, conic = np.zeros((n, 2)), np.zeros((n, 3)), np.zeros((n, 3))
        radius, depth, alpha = np.zeros(n), np.zeros(n), np.zeros(n)
        color, t = np.zeros((n, 3)), np.zeros((n, 3))
        lib.oracle_frame_projections(h, _ptr(gid, _ip), _ptr(p), _ptr(cov), _ptr(conic), _ptr(radius),
                                     _ptr(depth), _ptr(color), _ptr(alpha), _ptr(t))
        tx, ty = C.c_int(0), C.c_int(0)
        m = lib.oracle_frame_tile_count(h, C.byref(tx), C.byref(ty))
        offsets = np.zeros(tx.value * ty.value + 1, dtype=np.int64)
        items = np.zeros(max(m, 1), dtype=np.int32)
        lib.oracle_frame_tile_lists(h, _ptr(offsets, _lp), _ptr(items, _ip))
        items = items[:m]
        rgb = np.zeros((H, W, 3))
        T = np.zeros((H, W))
        con = np.zeros((H, W), dtype=np.int32)
        last = np.zeros((H, W), dtype=np.int32)
        lib.oracle_frame_pixels(h, _ptr(rgb), _ptr(T), _ptr(con, _ip), _ptr(last, _ip))
        return Frame(W, H, gid, p, cov, conic, radius, depth, color, alpha, t, tx.value, ty.value,
                     offsets, items, rgb, T, con, last, h if keep_handle else None)

    def free(self, frame: Frame):
        if frame.handle:
            self.lib.oracle_frame_free(frame.handle)
            frame.handle = None

    def backward(self, frame: Frame, d_image, cloud, pose, grads: Grads | None = None) -> Grads:
        assert frame.handle, "render with keep_handle=True"
        if grads is None:
            grads = Grads.zeros(cloud.n, cloud.basis_count)
        keep = []
        c = self._cloud(cloud, keep)
        di = np.ascontiguousarray(d_image, dtype=np.float64)
        pose = np.ascontiguousarray(pose, dtype=np.float64)
        g = _Grads(_ptr(grads.d_position), _ptr(grads.d_sh), _ptr(grads.d_rotation),
                   _ptr(grads.d_log_scale), _ptr(grads.d_opacity_logit), _ptr(grads.d_screen),
                   _ptr(grads.screen_norm_sum), _ptr(grads.screen_hits, _lp))
        rc = self.lib.oracle_backward(frame.handle, _ptr(di), C.byref(c), _ptr(pose), frame.width,
                                      frame.height, C.byref(g))
        if rc != 0:
            raise ValueError("StateMismatch: render output does not match the given scene")
        return grads

    def adam_step(self, cloud, grads: Grads, state: AdamState, cfg: AdamConfig, extent: float,
                  iteration: int):
        """Mutates ``cloud`` (float64 arrays in place) and ``state``."""
        for a in (cloud.positions, cloud.sh, cloud.rotations, cloud.log_scales, cloud.opacity_logits):
            assert a.dtype == np.float64 and a.flags.c_contiguous
        keep = []
        c = self._cloud(cloud, keep)
        g = _Grads(_ptr(grads.d_position), _ptr(grads.d_sh), _ptr(grads.d_rotation),
                   _ptr(grads.d_log_scale), _ptr(grads.d_opacity_logit), _ptr(grads.d_screen),
                   _ptr(grads.screen_norm_sum), _ptr(grads.screen_hits, _lp))
        s = _Adam(*[_ptr(getattr(state, f)) for f in
                    ("m_position", "v_position", "m_sh", "v_sh", "m_rotation", "v_rotation",
                     "m_scale", "v_scale", "m_opacity", "v_opacity")], state.step)
        k = _AdamCfg(cfg.iterations, cfg.lr_position_init, cfg.lr_position_final, cfg.lr_sh_dc,
                     cfg.lr_sh_rest, cfg.lr_opacity, cfg.lr_scale, cfg.lr_rotation)
        self.lib.oracle_adam_step(C.byref(c), C.byref(g), C.byref(s), C.byref(k), extent, iteration)
        state.step = s.step

    def loss(self, rendered, gt, lambda_ssim=0.2, mask_bottom_fraction=0.0):
        r = np.ascontiguousarray(rendered, dtype=np.float64)
        g = np.ascontiguousarray(gt, dtype=np.float64)
        H, W = r.shape[:2]
        d = np.zeros_like(r)
        v = self.lib.oracle_loss(_ptr(r), _ptr(g), W, H, lambda_ssim, mask_bottom_fraction, _ptr(d))
        return v, d

    def metrics(self, a, b):
        """(psnr, ssim) of two H x W x 3 images (metrics.cpp:64-79, osplat_metrics)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        assert a.shape == b.shape and a.ndim == 3 and a.shape[2] == 3
        ps, ss = C.c_double(0.0), C.c_double(0.0)
        self.lib.oracle_metrics(_ptr(a), _ptr(b), a.shape[1], a.shape[0], C.byref(ps), C.byref(ss))
        return ps.value, ss.value

    def cube_crops(self, pano, size: int):
        """The 6 cube-face perspective crops (eval.cpp:10-61) of an H x W x 3 panorama; reference only."""
        pano = np.ascontiguousarray(pano, dtype=np.float64)
        out = np.zeros((6, size, size, 3))
        fn = self.lib.oracle_ref_cube_crops
        fn.argtypes, fn.restype = [_dp, C.c_int, C.c_int, C.c_int, _dp], None
        fn(_ptr(pano), pano.shape[1], pano.shape[0], size, _ptr(out))
        return out

    def densify_and_prune(self, cloud, norm_sum, hits, max_radius, state: AdamState, cfg: DensifyConfig,
                          extent: float, seed: int, radius_prune_active: bool):
        """densify_and_prune (trainer.cpp:188-275) -> (new cloud, new AdamState, summary dict)."""
        import copy
        n, bc = cloud.n, cloud.basis_count
        keep = []
        c = self._cloud(cloud, keep)
        ns = np.ascontiguousarray(norm_sum, dtype=np.float64)
        hi = np.ascontiguousarray(hits, dtype=np.int64)
        mr = np.ascontiguousarray(max_radius, dtype=np.float64)
        cap = max(3 * n, 1)
        out = cloud.copy()
        out.positions, out.sh = np.zeros((cap, 3)), np.zeros((cap, bc, 3))
        out.rotations, out.log_scales, out.opacity_logits = np.zeros((cap, 4)), np.zeros((cap, 3)), np.zeros(cap)
        oc = _Cloud(0, cloud.sh_degree, cloud.active_sh_degree,
                    *[_ptr(a) for a in (out.positions, out.sh, out.rotations, out.log_scales, out.opacity_logits)])
        sin = [np.ascontiguousarray(getattr(state, f), dtype=np.float64) for f in ADAM_FIELDS]
        s_in = _Adam(*[_ptr(a) for a in sin], state.step)
        so = AdamState.zeros(cap, bc)
        s_out = _Adam(*[_ptr(getattr(so, f)) for f in ADAM_FIELDS], 0)
        k = _DensifyCfg(*[getattr(cfg, f) for f, _ in _DensifyCfg._fields_])
        e = _Edit()
        self.lib.oracle_densify_and_prune(C.byref(c), _ptr(ns), _ptr(hi, _lp), _ptr(mr), C.byref(s_in), C.byref(k),
                                          float(extent), C.c_ulonglong(seed), int(bool(radius_prune_active)),
                                          C.byref(oc), C.byref(s_out), C.byref(e))
        m = oc.n
        out.positions, out.sh, out.rotations = out.positions[:m].copy(), out.sh[:m].copy(), out.rotations[:m].copy()
        out.log_scales, out.opacity_logits = out.log_scales[:m].copy(), out.opacity_logits[:m].copy()
        for f in ADAM_FIELDS:
            setattr(so, f, getattr(so, f)[:m].copy())
        so.step = s_out.step
        return out, so, {"cloned": e.cloned, "split": e.split, "pruned": e.pruned, "final_count": e.final_count}

    def reset_opacity(self, cloud, ceiling: float):
        """reset_opacity (trainer.cpp:277-280); mutates cloud.opacity_logits in place."""
        assert cloud.opacity_logits.dtype == np.float64 and cloud.opacity_logits.flags.c_contiguous
        keep = []
        c = self._cloud(cloud, keep)
        c.opacity_logits = _ptr(cloud.opacity_logits)
        self.lib.oracle_reset_opacity(C.byref(c), float(ceiling))

    def mix64(self, x: int) -> int:
        return int(self.lib.oracle_mix64(C.c_ulonglong(x & 0xFFFFFFFFFFFFFFFF)))

    def save_checkpoint(self, cloud, path: str):
        """Reference save_checkpoint (dataio.cpp:347-382); reference library only."""
        keep = []
        c = self._cloud(cloud, keep)
        fn = self.lib.oracle_ref_save_checkpoint
        fn.argtypes, fn.restype = [C.POINTER(_Cloud), C.c_char_p], C.c_int
        assert fn(C.byref(c), path.encode()) == 0

    def save_optimizer_state(self, state: AdamState, n: int, bc: int, iteration: int, path: str):
        """Reference save_optimizer_state (dataio.cpp:479-495); reference library only."""
        arrs = [np.ascontiguousarray(getattr(state, f), dtype=np.float64) for f in ADAM_FIELDS]
        s = _Adam(*[_ptr(a) for a in arrs], state.step)
        fn = self.lib.oracle_ref_save_optimizer_state
        fn.argtypes, fn.restype = [C.POINTER(_Adam), C.c_int, C.c_int, C.c_long, C.c_char_p], C.c_int
        assert fn(C.byref(s), n, bc, iteration, path.encode()) == 0

    def mt64_draws(self, seed: int, count: int) -> list:
        out = (C.c_ulonglong * max(count, 1))()
        self.lib.oracle_mt64_draws(C.c_ulonglong(seed & 0xFFFFFFFFFFFFFFFF), count, out)
        return [int(out[i]) for i in range(count)]

    def epoch_order(self, train_indices, seed: int, epoch: int) -> list:
        """Trainer::pick_view's per-epoch Fisher-Yates shuffle (trainer.cpp:340-352)."""
        order = list(train_indices)
        draws = self.mt64_draws(self.mix64(seed ^ self.mix64(epoch)), max(len(order) - 1, 0))
        for k, i in enumerate(range(len(order), 1, -1)):
            j = draws[k] % i
            order[i - 1], order[j] = order[j], order[i - 1]
        return order


def load(kind: str = "port") -> Oracle:
    return Oracle(kind)


def available(kind: str) -> bool:
    return os.path.exists(PATHS[kind])
