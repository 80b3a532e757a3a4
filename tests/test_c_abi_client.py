"""The C ABI is consumable from plain C: compile tests/c_abi_client.c with gcc against
include/osplat.h, link libosplat_b200.so, run it (host-only here; + GPU render/train on a GPU box)."""
import os
import subprocess

import pytest

from paper_2404_03202_b200 import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "c_abi_client")
    libdir = os.path.dirname(native.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_abi_client.c"), "-o", exe, "-L", libdir, "-l:libosplat_b200.so",
                    f"-Wl,-rpath,{libdir}", "-lm"], check=True)
    return exe


def test_c_client_host_calls(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "cpu", str(tmp_path / "c.ply")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "version 0.1.0" in r.stdout and r.stdout.strip().endswith("ok")
    assert "last_error ParseError: unknown config key: nope" in r.stdout


@pytest.mark.gpu
def test_c_client_gpu_calls(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu", str(tmp_path / "c.ply")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "render sum" in r.stdout and r.stdout.strip().endswith("ok")
