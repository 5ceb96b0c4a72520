"""The drop-in boundary from plain C: examples/c_abi_demo.c is compiled with
gcc against include/lattdse_c.h and linked to the in-tree library, the way a
C/cgo/JNI consumer would. CPU part: lattice hash of the
reference Fig. 1 lattice, error-code mapping, CBC + anti-aliasing. GPU part:
64 Strang steps with unit-norm check."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PKG = os.path.join(ROOT, "paper_1808_06357_b200")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cabi") / "c_abi_demo")
    subprocess.run(
        ["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
         os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", PKG, "-llattdse_b200",
         f"-Wl,-rpath,{PKG}", "-lm", "-o", out],
        check=True)
    return out


def test_c_consumer_cpu(demo):
    r = subprocess.run([demo], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fig1 hash=0xc52fc32f65226f72" in r.stdout
    assert "C0 z=(1,1588)" in r.stdout


@pytest.mark.gpu
def test_c_consumer_gpu(demo):
    r = subprocess.run([demo, "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "64 Strang steps" in r.stdout
