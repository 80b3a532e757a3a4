"""GPU: the library's own data plane at world 2 on the one GPU of the box. The two ranks are two
contexts driven by two host threads in one process, their collectives carried by the in-process NCCL
stand-in tests/mock_nccl (loaded through OSPLAT_NCCL_LIB): sharded Adam steps and a densify exchange
equal the single-process batch computation bit for bit, and osplat_gpu_train at world 2 leaves both
ranks with identical parameters (tests/mock_nccl/world2_check.py)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
MOCK = os.path.join(HERE, "mock_nccl", "libmock_nccl.so")


@pytest.fixture(scope="module")
def world2():
    if not os.path.exists(MOCK):
        subprocess.run(["make", "-C", os.path.dirname(MOCK)], check=True, capture_output=True)
    env = dict(os.environ, OSPLAT_NCCL_LIB=MOCK)
    p = subprocess.run([sys.executable, os.path.join(HERE, "mock_nccl", "world2_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_world2_sharded_steps_and_densify_match_single_process(world2):
    r = world2["dp_steps"]
    s = r["ref_summary"]
    assert s["cloned"] + s["split"] > 0, s  # the densify iteration edits the set
    assert r["rank_summaries"] == [s, s], r
    assert r["n"] == [r["ref_n"]] * 2
    assert r["identical_to_single_process"], r["max_abs_diff"]


def test_world2_osplat_gpu_train_replicas_identical(world2):
    r = world2["train"]
    assert r["ranks_identical"], r
    assert "final.ply" in r["rank0_files"] and "metrics.jsonl" in r["rank0_files"], r
    assert r["rank1_files"] == [] or "final.ply" not in r["rank1_files"], r  # rank 0 writes the files
