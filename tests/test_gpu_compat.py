"""GPU: drop-in at the reference's C++ API and on host projection records.

* The reference's own tests/test_rasterizer.cpp, compiled unmodified against
  paper_2404_03202_b200/compat/rasterizer_gpu.cpp (which replaces proj/src/rasterizer.cpp), passes on
  the B200 — except three assertions that the FP32 parameter contract cannot meet and that are
  checked here to fail exactly where expected: 1e-9 / 1e-12 relative tolerances on values computed
  from FP64 parameters (cov of an FP64 sigma; an analytic value from FP64 opacity / colour), and the
  "1 instance" check that fails against the reference itself.
* osplat_gpu_render_projected (bin_to_tiles + blend_forward on host SplatProjection records) matches
  the oracle's restatement of those functions: tile lists and contributor counts bit-exact, image
  within IMAGE_ATOL, with device binning and with a caller-supplied grid.
* Feeding a frame's own records back reproduces the frame bit for bit.
"""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2404_03202_b200 import native, scenes

from parity import IMAGE_ATOL
from splat_records import random_splats

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPAT_BIN = os.path.join(ROOT, "oracle", "_ref", "compat", "test_rasterizer_gpu")
# test case -> the assertion lines (proj/tests/test_rasterizer.cpp) allowed to fail, and why
EXPECTED_FAILURES = {
    "project_gaussian on the optical axis": {44, 45},  # cov.a/c vs FP64 sigma at 1e-9 (FP32 log-scale)
    "bin_to_tiles basics and seam wrap": {80},  # fails against the reference itself (boundary splat)
    "reference_render reproduces the analytic single-splat value": {206},  # 1e-12 vs FP64 opacity/colour
}


def _run(*args):
    if not os.path.exists(COMPAT_BIN):
        pytest.fail(f"{COMPAT_BIN} not built (make -C oracle compat-tests, needs the reference tree)")
    return subprocess.run([COMPAT_BIN, *args], capture_output=True, text=True, timeout=600)


def test_reference_rasterizer_suite_on_gpu():
    r = _run("-tce=" + ",".join(EXPECTED_FAILURES))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 8 passed | 0 failed" in r.stdout, r.stdout


def test_reference_rasterizer_expected_failures_only():
    r = _run()
    out = r.stdout + r.stderr
    failed_cases = set(re.findall(r"^\[FAIL\] (.*)$", out, re.M))
    assert failed_cases <= set(EXPECTED_FAILURES), out
    lines = {int(x) for x in re.findall(r"test_rasterizer\.cpp:(\d+): CHECK FAILED", out)}
    allowed = set().union(*EXPECTED_FAILURES.values())
    assert lines <= allowed, (lines, out)
    assert "exception" not in out, out


@pytest.mark.parametrize("n,W,H,seed", [(0, 64, 32, 0), (1, 64, 32, 1), (60, 128, 64, 2), (400, 256, 128, 3),
                                        (3000, 512, 256, 4)])
def test_render_projected_matches_oracle(oracle_port, n, W, H, seed):
    s = random_splats(n, W, H, seed)
    bg = (0.2, 0.3, 0.4)
    ctx = native.Context(scenes.synthetic_cloud(1, seed=0))
    of = oracle_port.blend_projections(s, W, H, bg)
    fr = ctx.render_projected(s, W, H, bg)
    tx, ty, ranges, ids = fr.tiles()
    assert (tx, ty) == (of.tiles_x, of.tiles_y)
    for t in range(tx * ty):
        assert np.array_equal(ids[ranges[t, 0]:ranges[t, 1]], of.items[of.offsets[t]:of.offsets[t + 1]]), t
    rgb, T, con, last = fr.pixels()
    assert np.array_equal(con, of.contributors) and np.array_equal(last, of.last_contrib)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
    assert np.max(np.abs(T - of.T)) <= IMAGE_ATOL
    # a caller-supplied grid (every list reversed) is blended as given
    rev = [of.items[of.offsets[t]:of.offsets[t + 1]][::-1] for t in range(tx * ty)]
    offs = np.concatenate([[0], np.cumsum([len(x) for x in rev])]).astype(np.int64)
    items = np.concatenate(rev + [np.zeros(0, dtype=np.int32)]).astype(np.int32)
    of2 = oracle_port.blend_projections(s, W, H, bg, grid=(offs, items))
    fr2 = ctx.render_projected(s, W, H, bg, grid=(np.stack([offs[:-1], offs[1:]], 1), items))
    _, T2, con2, last2 = fr2.pixels()
    assert np.array_equal(con2, of2.contributors) and np.array_equal(last2, of2.last_contrib)
    assert np.max(np.abs(fr2.image() - of2.rgb)) <= IMAGE_ATOL
    sp = fr.splats()
    for k in ("gaussian_id", "p", "cov", "conic", "radius", "depth", "color", "alpha_base"):
        assert np.array_equal(sp[k], np.asarray(s[k], dtype=sp[k].dtype)), k


def test_frame_records_round_trip():
    """render -> osplat_frame_splats -> render_projected reproduces the frame exactly."""
    cloud = scenes.synthetic_cloud(20000, seed=5)
    pose = scenes.ring_poses(4, seed=2)[1]
    W, H = 512, 256
    ctx = native.Context(cloud)
    fr = ctx.render(pose, W, H, (0.1, 0.0, 0.3))
    sp = fr.splats()
    vis = fr.projections()["visible"]
    assert np.array_equal(sp["gaussian_id"], np.nonzero(vis)[0])
    fp = ctx.render_projected(sp, W, H, (0.1, 0.0, 0.3))
    a, b = fr.pixels(), fp.pixels()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    _, _, r1, i1 = fr.tiles()
    _, _, r2, i2 = fp.tiles()
    assert np.array_equal(r1, r2)
    assert np.array_equal(i1, sp["gaussian_id"][i2])  # record index -> Gaussian id


def test_projected_frame_has_no_backward():
    ctx = native.Context(scenes.synthetic_cloud(100, seed=1))
    s = random_splats(10, 64, 32, 9)
    fr = ctx.render_projected(s, 64, 32)
    with pytest.raises(native.OsplatError) as e:
        ctx.backward(fr, np.zeros((32, 64, 3)))
    assert "StateMismatch" in str(e.value)
    bad = dict(s, depth=np.full(10, -1.0))
    with pytest.raises(native.OsplatError):
        ctx.render_projected(bad, 64, 32)


def test_render_projected_edge_records(oracle_port):
    """Records the reference bins but never blends (alpha_base < 1/255), records at and across the
    seam (centre outside [0, W)), a full-width record (span >= tiles_x), equal (depth, id) pairs, and
    a zero-radius record: tile lists and pixels as bin_to_tiles + blend_forward give them."""
    W, H = 128, 64
    s = random_splats(40, W, H, 31)
    s["alpha_base"][:5] = 1.0 / 300.0                 # below 1/255: binned, never blended
    s["p"][5] = (-0.75, 20.0)                          # left of the seam
    s["p"][6] = (W + 0.3, 40.0)                        # right of the seam
    s["p"][7] = (W * 0.5, 3.0)
    s["radius"][7] = 3.0 * W                           # wider than the image: whole rows
    s["depth"][8] = s["depth"][9]
    s["gaussian_id"][8] = s["gaussian_id"][9]          # full (depth, id) tie: any order is the reference's
    s["radius"][10] = 0.0
    ctx = native.Context(scenes.synthetic_cloud(1, seed=0))
    of = oracle_port.blend_projections(s, W, H)
    fr = ctx.render_projected(s, W, H)
    tx, ty, ranges, ids = fr.tiles()
    for t in range(tx * ty):
        g = ids[ranges[t, 0]:ranges[t, 1]]
        o = of.items[of.offsets[t]:of.offsets[t + 1]]
        assert len(g) == len(o), t
        # equal (depth, id) records may come in either order; everything else matches exactly
        key = lambda i: (s["depth"][i], s["gaussian_id"][i])
        assert [key(i) for i in g] == [key(i) for i in o], t
    rgb, T, con, last = fr.pixels()
    assert np.array_equal(con, of.contributors) and np.array_equal(last, of.last_contrib)
    assert np.max(np.abs(fr.image() - of.rgb)) <= IMAGE_ATOL
