"""The C-ABI boundary (include/lattdse_c.h) and host logic, CPU only:
library loads, every declared symbol is exported, error codes map 1:1 to
lattdse::Errc (errors.hpp:8-22), the seed schedule matches an independent
restatement, and the pass-kernel emulation (index algebra of every program)
is exact against naive DFTs."""
import ctypes
import math
import os
import subprocess

import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(L.LIB_PATH)
    syms = L.exported_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert "sm_100a" in L.version()


def test_error_codes_map_to_errc_ordinals():
    lib = ctypes.CDLL(L.LIB_PATH)
    lib.lattdse_last_error.restype = ctypes.c_char_p
    out = ctypes.c_void_p()
    gen = (ctypes.c_int64 * 4)(1, 0, 0, 1)
    mod = (ctypes.c_int64 * 2)(4, 8)
    rc = lib.lattdse_lattice_create(2, 2, gen, mod, ctypes.byref(out))
    assert rc == 2  # non_divisible_moduli = ordinal 1 -> code 2
    assert b"does not divide" in lib.lattdse_last_error()
    assert lib.lattdse_last_error_code() == 2
    rc = lib.lattdse_lattice_create(2, 1, None, mod, ctypes.byref(out))
    assert rc == 1  # NULL -> invalid_argument, no crash
    rc = lib.lattdse_lattice_from_json(b"{bad", ctypes.byref(out))
    assert rc == 13  # io_error
    assert L.ERRC[13] == "device_error" and L.ERRC[14] == "unsupported"


def test_solver_without_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    lat = L.Lattice.rank1([1, 34], 55)
    a, b, c, p = L.problem_draw(1, 2, 1, 0.4, 0.6, 2)
    with pytest.raises(L.LattdseError) as e:
        L.Solver(lat, 0.1, a, b, c, p, 0.1)
    assert e.value.name == "device_error"


class SplitMix64:
    """Independent restatement of the documented seed schedule."""

    def __init__(self, seed):
        self.s = seed & 0xFFFFFFFFFFFFFFFF

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def uniform(self, lo=0.0, hi=1.0):
        return lo + (hi - lo) * ((self.next() >> 11) * 2.0 ** -53)

    def integer(self, lo, hi):
        return lo + min(int(math.floor(self.uniform() * (hi - lo + 1))), hi - lo)


@pytest.mark.parametrize("name", ["C0", "C1", "C2", "C3", "C4"])
def test_seed_schedule(name):
    cfg = configs.CONFIGS[name]
    a, b, c, p = configs.problem(cfg, batch=min(cfg.batch, 3))
    r = SplitMix64(cfg.seed)
    d = cfg.d
    assert np.array_equal(a, [r.uniform(0.5, 1.5) for _ in range(d)])
    assert np.array_equal(b, [r.uniform(0.0, 0.5) for _ in range(d - 1)])
    lo, hi = cfg.c_range
    if cfg.batch == 1:
        assert np.array_equal(c[0], [r.uniform(lo, hi) for _ in range(d)])
        assert np.array_equal(p[0], [r.integer(-cfg.p_max, cfg.p_max) for _ in range(d)])
    else:
        for m in range(c.shape[0]):
            rm = SplitMix64(SplitMix64(cfg.seed ^ (m + 1)).next())
            assert np.array_equal(c[m], [rm.uniform(lo, hi) for _ in range(d)])
            assert np.array_equal(p[m], [rm.integer(-cfg.p_max, cfg.p_max) for _ in range(d)])
    assert np.all((a >= 0.5) & (a < 1.5)) and np.all((b >= 0) & (b < 0.5))
    assert np.all(np.abs(p) <= cfg.p_max)


def test_shard_members_partition():
    for batch in (1, 7, 512):
        for world in (1, 2, 3, 8):
            seen = []
            for rank in range(world):
                m0, cnt = configs.shard_members(batch, rank, world)
                seen.extend(range(m0, m0 + cnt))
            assert seen == list(range(batch))


def test_pass_kernel_emulation():
    """nvcc-built host harness: every pass program of the generic kernels
    (four-step and Good-Thomas layouts) vs naive long-double DFTs."""
    exe = os.path.join(ROOT, "paper_1808_06357_b200", "csrc", "build", "fft_hosttest")
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1808_06357_b200", "csrc"), "hosttest"], check=True,
                   stdout=subprocess.DEVNULL)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ALL OK" in out.stdout, out.stdout[-2000:]


def test_lean_kernel_launch_geometry():
    """Compile-time launch geometry of the lean per-step kernels for the lengths
    the five configs run (pass_instantiate.cuh Geometry4): the measured choices
    of profiles/r2/p4_sweep*.txt, and which plans take the swizzled slots."""
    csrc = os.path.join(ROOT, "paper_1808_06357_b200", "csrc")
    subprocess.run(["make", "-C", csrc, "geomtest"], check=True, stdout=subprocess.DEVNULL)
    out = subprocess.run([os.path.join(csrc, "build", "pass4_geomtest")], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    rows = {int(line.split()[0][2:]): line for line in out.stdout.splitlines() if line.startswith("L=")}
    # config 3: COL 486 four columns in place, 4 CTAs of 224 threads (+ the eight-column variant); ROW 1080 (9,12,10) in place, 6 CTAs of 128
    assert "plan 9 9 6 ok=1 swz=0" in rows[486] and "COL B=4 pp=0 NT=224 MB=4" in rows[486] and "WIDE ok=1 B=8 NT=448 MB=2" in rows[486]
    assert "plan 9 12 10 ok=1 swz=0" in rows[1080] and "ROW B=1 pp=0 NT=128 MB=6" in rows[1080]
    # config 1: COL 1296 two columns with two stage buffers; ROW 1620 two buffers at 3 CTAs
    assert "COL B=2 pp=1 NT=288 MB=2" in rows[1296] and "ROW B=1 pp=1 NT=192 MB=3" in rows[1620]
    # power-of-two plans run swizzled (config 2's 4096, config 4's 2048-long rows); 512 / 1024 stay on the generic kernels
    assert "ok=1 swz=1" in rows[4096] and "ROW B=1 pp=0 NT=256 MB=2" in rows[4096] and "COL B=2 pp=0 NT=512 MB=1" in rows[4096]
    assert "ok=1 swz=1" in rows[2048] and "ROW B=1 pp=0 NT=128 MB=4" in rows[2048]
    assert "ok=0" in rows[512] and "ok=0" in rows[1024]
