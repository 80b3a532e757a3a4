"""CPU: pin the C restatement of densify_and_prune / reset_opacity / the trainer RNG
(oracle/oracle.c) against the reference's own trainer.cpp (oracle/_ref). Bit-identical outputs:
both use FP64 in the reference's operation order, and the port's mt19937_64 + polar normal
restatement must reproduce libstdc++'s std::normal_distribution stream exactly.
"""
import numpy as np
import pytest

import pyoracle
from paper_2404_03202_b200 import scenes


def densify_inputs(n, seed, split_heavy=False):
    """A cloud plus screen statistics that exercise clone, split and every prune rule."""
    rng = np.random.default_rng(seed)
    cloud = scenes.synthetic_cloud(n, seed=seed)
    # spread of world scales across the split threshold (0.01 * extent) and the prune threshold
    ls = np.log(rng.uniform(0.002, 0.05 if split_heavy else 0.02, size=(n, 3)))
    ls[rng.random(n) < 0.02] = np.log(0.2)  # oversized -> world-scale prune
    cloud.log_scales = ls.astype(np.float32).astype(np.float64)
    op = cloud.opacity_logits.copy()
    op[rng.random(n) < 0.05] = -6.0  # sigmoid < 0.005 -> opacity prune
    cloud.opacity_logits = op.astype(np.float32).astype(np.float64)
    hits = rng.integers(0, 5, size=n).astype(np.int64)
    norm_sum = rng.uniform(0, 8e-4, size=n) * hits
    max_radius = np.floor(rng.uniform(0, 40, size=n))
    st = pyoracle.AdamState.zeros(n, cloud.basis_count)
    for f in pyoracle.ADAM_FIELDS:
        setattr(st, f, rng.standard_normal(getattr(st, f).shape) * 1e-3)
    st.step = 17
    return cloud, norm_sum, hits, max_radius, st


@pytest.mark.parametrize("n,seed,radius_active,split_heavy", [(500, 1, False, False), (2000, 2, True, False),
                                                             (1500, 3, True, True), (0, 4, True, False)])
def test_densify_port_bit_exact_vs_reference(n, seed, radius_active, split_heavy, oracle_port, oracle_ref):
    cloud, ns, hits, mr, st = densify_inputs(max(n, 1), seed, split_heavy)
    if n == 0:
        cloud = scenes.Cloud(np.zeros((0, 3)), np.zeros((0, 16, 3)), np.zeros((0, 4)), np.zeros((0, 3)),
                             np.zeros(0))
        ns, hits, mr = np.zeros(0), np.zeros(0, dtype=np.int64), np.zeros(0)
        st = pyoracle.AdamState.zeros(0, 16)
    cfg = pyoracle.DensifyConfig()
    rng_seed = oracle_ref.mix64(123 ^ oracle_ref.mix64(0x5EED + 500))
    a = oracle_port.densify_and_prune(cloud, ns, hits, mr, st, cfg, 1.0, rng_seed, radius_active)
    b = oracle_ref.densify_and_prune(cloud, ns, hits, mr, st, cfg, 1.0, rng_seed, radius_active)
    assert a[2] == b[2]
    if n:
        assert a[2]["cloned"] > 0 and a[2]["split"] > 0 and a[2]["pruned"] > 0
    for f in ("positions", "sh", "rotations", "log_scales", "opacity_logits"):
        assert np.array_equal(getattr(a[0], f), getattr(b[0], f)), f
    for f in pyoracle.ADAM_FIELDS:
        assert np.array_equal(getattr(a[1], f), getattr(b[1], f)), f
    assert a[1].step == b[1].step == st.step


def test_mix64_and_reset_opacity(oracle_port, oracle_ref):
    for x in (0, 1, 0x5EED, 2**63 + 12345, 2**64 - 1):
        assert oracle_port.mix64(x) == oracle_ref.mix64(x)
    cloud = scenes.synthetic_cloud(300, seed=9)
    a, b = cloud.copy(), cloud.copy()
    oracle_port.reset_opacity(a, 0.01)
    oracle_ref.reset_opacity(b, 0.01)
    assert np.array_equal(a.opacity_logits, b.opacity_logits)
    assert np.max(a.opacity_logits) == np.log(0.01 / 0.99)


def test_mt64_stream_and_epoch_order(oracle_port, oracle_ref):
    for seed in (0, 5489, 2**64 - 3):
        assert oracle_port.mt64_draws(seed, 700) == oracle_ref.mt64_draws(seed, 700)
    assert oracle_port.mt64_draws(5489, 1) == [14514284786278117030]  # std::mt19937_64 default-seed value
    order = oracle_port.epoch_order(list(range(10)), 7, 3)
    assert sorted(order) == list(range(10)) and order == oracle_ref.epoch_order(list(range(10)), 7, 3)
