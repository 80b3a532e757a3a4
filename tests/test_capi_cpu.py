"""CPU: the C-ABI library loads, exports every symbol include/osplat.h declares, and the host-side
logic (error mapping, cloud handles, checkpoint PLY, config) behaves like the reference's capi.cpp.
No kernel is launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "osplat.h")

# The reference C ABI entry points on this path (proj/include/omnisplat/capi.h:31-88).
REFERENCE_SYMBOLS = ["osplat_version", "osplat_last_error", "osplat_set_threads", "osplat_cloud_load",
                     "osplat_cloud_save", "osplat_cloud_count", "osplat_cloud_free", "osplat_config_create",
                     "osplat_config_set", "osplat_config_free", "osplat_render", "osplat_image_width",
                     "osplat_image_height", "osplat_image_pixels", "osplat_image_free", "osplat_metrics",
                     "osplat_report_view_count", "osplat_report_view", "osplat_report_mean", "osplat_report_mode",
                     "osplat_report_free"]


def declared_symbols():
    text = open(HEADER).read()
    return re.findall(r"^OSPLAT_API [^(]*?\b(osplat_\w+)\(", text, flags=re.M)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_reference_symbols_present_in_header():
    syms = set(declared_symbols())
    assert set(REFERENCE_SYMBOLS) <= syms


def test_version_and_status_codes():
    assert native.version() == "0.1.0"
    text = open(HEADER).read()
    for name, val in [("OSPLAT_OK", 0), ("OSPLAT_ERR_INVALID_ARGUMENT", 1), ("OSPLAT_ERR_IO", 2),
                      ("OSPLAT_ERR_PARSE", 3), ("OSPLAT_ERR_VALIDATION", 4), ("OSPLAT_ERR_UNSUPPORTED", 5),
                      ("OSPLAT_ERR_RUNTIME", 6)]:
        assert re.search(rf"{name} = {val}\b", text)


def test_cloud_roundtrip():
    cloud = scenes.synthetic_cloud(257, seed=3)
    cloud.active_sh_degree = 2
    hc = native.HostCloud.from_cloud(cloud)
    assert len(hc) == 257
    back = hc.to_cloud()
    for k in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
        assert np.array_equal(getattr(back, k), getattr(cloud, k))
    assert back.sh_degree == 3 and back.active_sh_degree == 2


def test_checkpoint_ply_roundtrip(tmp_path):
    """save_checkpoint / load_checkpoint format (dataio.cpp:347-453): float32 properties,
    f_rest channel-major, sh_degree comment; load sets active = sh_degree."""
    for deg in (0, 1, 3):
        cloud = scenes.random_cloud(np.random.default_rng(deg), count=33, sh_degree=deg)
        hc = native.HostCloud.from_cloud(cloud)
        path = str(tmp_path / f"c{deg}.ply")
        hc.save(path)
        raw = open(path, "rb").read()
        header = raw[:raw.index(b"end_header\n")].decode()
        assert header.startswith("ply\nformat binary_little_endian 1.0\ncomment format_version 1\n")
        assert f"comment sh_degree {deg}\nelement vertex 33\n" in header
        nrest = 3 * ((deg + 1) ** 2 - 1)
        props = re.findall(r"property float (\w+)", header)
        assert props[:9] == ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
        assert props[9:9 + nrest] == [f"f_rest_{i}" for i in range(nrest)]
        assert props[9 + nrest:] == ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
        back = native.HostCloud.load(path).to_cloud()
        for k in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
            assert np.array_equal(getattr(back, k), getattr(cloud, k)), (deg, k)
        assert back.sh_degree == deg and back.active_sh_degree == deg
        # channel-major f_rest: property f_rest_{c*(bc-1)+(j-1)} holds sh[j][c]
        if deg >= 1:
            body = np.frombuffer(raw[raw.index(b"end_header\n") + 11:], dtype="<f4").reshape(33, len(props))
            bc = (deg + 1) ** 2
            assert body[5, props.index("f_rest_0")] == np.float32(cloud.sh[5, 1, 0])
            assert body[5, props.index(f"f_rest_{bc - 1}")] == np.float32(cloud.sh[5, 1, 1])


def test_checkpoint_ply_bytes_match_reference_writer(tmp_path, oracle_ref):
    """Byte-identical to the reference's own save_checkpoint (dataio.cpp:347-382), and the
    reference file loads back bit-exactly through osplat_cloud_load."""
    for deg in (0, 2, 3):
        cloud = scenes.random_cloud(np.random.default_rng(10 + deg), count=41, sh_degree=deg)
        cloud.active_sh_degree = max(deg - 1, 0)
        ours, ref = str(tmp_path / f"o{deg}.ply"), str(tmp_path / f"r{deg}.ply")
        native.HostCloud.from_cloud(cloud).save(ours)
        oracle_ref.save_checkpoint(cloud, ref)
        assert open(ours, "rb").read() == open(ref, "rb").read(), deg
        back = native.HostCloud.load(ref).to_cloud()
        assert np.array_equal(back.sh, cloud.sh) and np.array_equal(back.positions, cloud.positions)


def test_checkpoint_errors(tmp_path):
    with pytest.raises(native.OsplatError) as e:
        native.HostCloud.load(str(tmp_path / "missing.ply"))
    assert e.value.status == native.IO and e.value.message.startswith("IoError: cannot open")
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"ply\nformat binary_little_endian 1.0\ncomment format_version 2\nend_header\n")
    with pytest.raises(native.OsplatError) as e:
        native.HostCloud.load(str(bad))
    assert e.value.status == native.UNSUPPORTED and "VersionMismatch" in e.value.message
    miss = tmp_path / "miss.ply"
    miss.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 0\nproperty float x\nend_header\n")
    with pytest.raises(native.OsplatError) as e:
        native.HostCloud.load(str(miss))
    assert e.value.status == native.PARSE and "MissingProperty" in e.value.message


def test_config_setters():
    cfg = native.Config(iterations=123, lr_sh_dc="0.01", seed=42)
    with pytest.raises(native.OsplatError) as e:
        cfg.set("no_such_key", 1)
    assert e.value.status == native.PARSE
    assert e.value.message == "ParseError: unknown config key: no_such_key"
    with pytest.raises(native.OsplatError) as e:
        cfg.set("iterations", "abc")
    assert e.value.status == native.PARSE and "is not a number" in e.value.message
    cfg.set("lambda_ssim", 0.0)
    assert native.lib.osplat_last_error().decode() == ""


def test_render_argument_errors():
    cloud = native.HostCloud.from_cloud(scenes.synthetic_cloud(10, seed=1))
    img = C.c_void_p()
    t = np.eye(4)
    st = native.lib.osplat_render(None, t.ctypes.data_as(native._dp), 64, 32, C.byref(img))
    assert st == native.INVALID_ARGUMENT
    assert native.lib.osplat_last_error().decode() == "osplat_render: null argument"
    st = native.lib.osplat_render(cloud.handle, t.ctypes.data_as(native._dp), 1, 32, C.byref(img))
    assert st == native.INVALID_ARGUMENT
    assert native.lib.osplat_last_error().decode() == "osplat_render: image size must be >= 2x2"
    skew = np.eye(4)
    skew[0, 1] = 0.01
    st = native.lib.osplat_render(cloud.handle, skew.ctypes.data_as(native._dp), 64, 32, C.byref(img))
    assert st == native.VALIDATION
    assert native.lib.osplat_last_error().decode() == "ValidationError: pose rotation is not orthonormal"
    mirrored = np.eye(4)
    mirrored[0, 0] = -1.0
    st = native.lib.osplat_render(cloud.handle, mirrored.ctypes.data_as(native._dp), 64, 32, C.byref(img))
    assert st == native.VALIDATION


def test_no_silent_cpu_fallback_without_gpu():
    """Without a CUDA device the product must fail loudly, never compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(native.OsplatError) as e:
        native.Context(scenes.synthetic_cloud(10, seed=1))
    assert e.value.status == native.RUNTIME and "CUDA" in e.value.message
    cloud = native.HostCloud.from_cloud(scenes.synthetic_cloud(10, seed=1))
    with pytest.raises(native.OsplatError):
        native.osplat_render(cloud, scenes.identity_pose(), 64, 32)


def test_loss_value_from_sums_is_the_reference_formula():
    """osplat_loss_value (host): (1 - l) L1/n + l (1 - mean SSIM) with the bottom-row mask
    (trainer.cpp:54-63), from the device's four sums {sum |r - g|, SSIM sums r, g, b}."""
    from paper_2404_03202_b200 import native
    W, H = 64, 32
    sums = np.array([123.25, 1500.5, 1490.0, 1510.75])
    for lam, mask in ((0.0, 0.0), (0.2, 0.0), (0.2, 0.25), (1.0, 0.1)):
        keep = H - int(np.floor(mask * H))
        npx = W * keep
        ref = (1 - lam) * sums[0] / (3 * npx)
        if lam > 0:
            ref += lam * (1 - (sums[1:].sum() / npx) / 3)
        assert native.loss_value(sums, lam, W, H, mask) == pytest.approx(ref, rel=1e-15, abs=1e-15)
