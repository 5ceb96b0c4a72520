"""The C++ drop-in boundary: examples/cxx_consumer.cpp, written against the
reference's public header (include/lattdse/lattice.hpp = lattice.hpp:17-86)
plus solver.hpp / setup.hpp / errors.hpp, compiled with g++ -std=c++20 and
linked to the in-tree library, as a reference C++ caller would be."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
PKG = os.path.join(ROOT, "paper_1808_06357_b200")


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cxx") / "cxx_consumer")
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cxx_consumer.cpp"), "-L", PKG, "-llattdse_b200",
                    f"-Wl,-rpath,{PKG}", "-o", out], check=True)
    return out


def test_cxx_consumer_cpu(demo):
    r = subprocess.run([demo], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fig1 hash=0xc52fc32f65226f72" in r.stdout
    assert "C0 z=(1,1588)" in r.stdout and "caught" in r.stdout and "cpu ok" in r.stdout


@pytest.mark.gpu
def test_cxx_consumer_gpu(demo):
    r = subprocess.run([demo, "--gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu ok" in r.stdout
