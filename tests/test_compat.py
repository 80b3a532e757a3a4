"""CPU: the host-projection oracle entry (oracle_blend_projections = bin_to_tiles + blend_forward on
host SplatProjection records) pinned against the reference's own functions, and the compat build
(the reference's test_rasterizer.cpp linked against paper_2404_03202_b200/compat) present and
bound to this library."""
import os
import subprocess

import numpy as np
import pytest

from splat_records import random_splats

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPAT_BIN = os.path.join(ROOT, "oracle", "_ref", "compat", "test_rasterizer_gpu")


@pytest.mark.parametrize("n,W,H,seed", [(0, 64, 32, 0), (1, 64, 32, 1), (60, 128, 64, 2), (400, 256, 128, 3)])
def test_blend_projections_port_matches_reference(oracle_port, oracle_ref, n, W, H, seed):
    s = random_splats(n, W, H, seed)
    bg = (0.2, 0.3, 0.4)
    a = oracle_port.blend_projections(s, W, H, bg)
    b = oracle_ref.blend_projections(s, W, H, bg)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.items, b.items)
    assert np.array_equal(a.rgb, b.rgb) and np.array_equal(a.T, b.T)
    assert np.array_equal(a.contributors, b.contributors) and np.array_equal(a.last_contrib, b.last_contrib)
    # a caller-supplied grid (every list reversed) is blended as given
    items = np.concatenate([a.items[a.offsets[t]:a.offsets[t + 1]][::-1] for t in range(len(a.offsets) - 1)]
                           + [np.zeros(0, dtype=np.int32)])
    a2 = oracle_port.blend_projections(s, W, H, bg, grid=(a.offsets, items))
    b2 = oracle_ref.blend_projections(s, W, H, bg, grid=(a.offsets, items))
    assert np.array_equal(a2.rgb, b2.rgb) and np.array_equal(a2.last_contrib, b2.last_contrib)
    assert np.array_equal(a2.items, items)


def test_compat_suite_is_built_against_this_library():
    if not os.path.exists("/root/reference/proj/tests/test_rasterizer.cpp") and not os.path.exists(COMPAT_BIN):
        pytest.skip("reference tree absent and no prebuilt compat suite")
    assert os.path.exists(COMPAT_BIN), "make -C oracle compat-tests"
    ldd = subprocess.run(["ldd", COMPAT_BIN], capture_output=True, text=True).stdout
    lib = os.path.join(ROOT, "paper_2404_03202_b200", "libosplat_b200.so")
    bound = [ln.split("=>")[1].split("(")[0].strip() for ln in ldd.splitlines() if "libosplat_b200.so =>" in ln]
    assert bound and os.path.realpath(bound[0]) == os.path.realpath(lib), ldd
    undef = subprocess.run(["nm", "-D", "--undefined-only", COMPAT_BIN], capture_output=True, text=True).stdout
    for sym in ("osplat_gpu_render", "osplat_gpu_render_projected", "osplat_frame_splats", "osplat_gpu_upload"):
        assert sym in undef, sym
    # the reference's CPU rasterizer is linked only for its brute-force reference_render
    syms = subprocess.run(["nm", "-C", COMPAT_BIN], capture_output=True, text=True).stdout
    assert "omnisplat::reference_render(" in syms
    assert "_cpu_oracle" in syms  # renamed reference definitions, not called by the suite
