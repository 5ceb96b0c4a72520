"""Full-run parity on the benched paths: the sm_100a solver (through the C
ABI) after 1 and after m Strang steps vs committed CPU-oracle fixtures
(tests/golden/run_<config>.npz, made by tests/golden/make_run_fixtures.py
from oracle/ alone: oracle/cases.py lattices and seeds, the oracle's own
shell-walk norm table, literal SPEC.md:336-344 steps).

Tolerances (BASELINE.json north_star): relative L2 <= 1e-12 after one step,
<= 1e-10 after the full run, | ||u|| - 1 | <= 1e-12. Each fixture holds a
seeded subset of coefficients (relative L2 over it) and four random-phase
linear functionals of the FULL coefficient vector (oracle/cases.checksums:
|S_k(e)| ~ ||e||, so they check the whole state). The norm table the solver
builds (device shell walk for rank 1, host walk for rank 2) must hash to the
oracle's: the index map is compared bit-exactly.

Config 3 runs the benched configuration itself: all 512 members in one
group (the 486 x 1080 ensemble geometry bench.py times), members 0, 255, 511
checked.
"""
import hashlib
import os

import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle.cases import checksums

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL_ONE, TOL_RUN, TOL_NORM = 1e-12, 1e-10, 1e-12


def fixture(name):
    path = os.path.join(GOLD, f"run_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return np.load(path)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check_state(got, fx, mi, tag, tol):
    idx = fx["idx"]
    want = fx[f"{tag}_{mi}"]
    assert rel(got[idx], want) <= tol, (tag, mi, rel(got[idx], want))
    cs = checksums(got)
    ref = fx[f"cs{tag[1:]}_{mi}"]
    scale = float(np.linalg.norm(got))
    assert np.max(np.abs(cs - ref)) <= 3 * tol * scale, (tag, mi, np.abs(cs - ref) / scale)


def solver_for(name, batch=None):
    cfg = configs.CONFIGS[name]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=batch)
    if cfg.rank == 1:
        norm2, _ = L.aaset_norms_device(lat)  # the table the solver itself uses (device shell walk)
        S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma)
    else:
        norm2, _, _ = L.aaset_build(lat, with_vectors=False)
        S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, norm2=norm2)
    S.set_dt(cfg.dt)
    S.discretize_initial()
    return cfg, S, np.ascontiguousarray(norm2, np.uint32)


@pytest.mark.parametrize("name", ["C0", "C1", "C2", "C3"])
def test_full_run_vs_oracle_fixture(name):
    fx = fixture(name)
    cfg, S, norm2 = solver_for(name)
    assert hashlib.sha256(norm2.tobytes()).digest() == fx["norm2_sha"].tobytes(), "norm table differs from oracle"
    assert S.n == int(fx["N"]) and cfg.m == int(fx["m"])
    members = [int(m) for m in fx["members"]]
    if name == "C3":
        info = S.info()
        assert S.batch == 512 and info["group"] == 512 and (info["M1"], info["M2"]) == (486, 1080), info
    S.step(1)
    for mi, mem in enumerate(members):
        got = S.get_state(L.COEFFICIENTS, m0=mem, count=1)[0]
        check_state(got, fx, mi, "u1", TOL_ONE)
    S.step(cfg.m - 1)
    norms, energies = S.l2_norm(), S.energy()
    for mi, mem in enumerate(members):
        got = S.get_state(L.COEFFICIENTS, m0=mem, count=1)[0]
        check_state(got, fx, mi, "um", TOL_RUN)
        assert abs(norms[mem] - 1.0) <= TOL_NORM
        # the oracle's own norm drifts by up to ~2e-12 over C1's 4096
        # recursive-FFT transforms (fixture nrmm 0.9999999999978751)
        assert abs(norms[mem] - float(fx[f"nrmm_{mi}"])) <= 1e-11
        e_ref = float(fx[f"enm_{mi}"])
        assert abs(energies[mem] - e_ref) <= 1e-10 * abs(e_ref)
    if name == "C3":
        # every member conserves its norm over the whole benched run
        assert np.max(np.abs(norms - 1.0)) <= TOL_NORM
