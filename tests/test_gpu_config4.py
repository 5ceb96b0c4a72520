"""Config 4 (d = 20, N = smallest prime >= 2^30) on ONE B200, and its
reduced-N twin C4r (N = smallest prime >= 2^24) against the oracle
(at full N the GPU is checked by invariants -- norm
conservation to 1e-12 and time-reversibility to 1e-10).

Both run the three-level layout (M = M1 x Ma x Mb), the device setup (norm
table, sampling) and, at full N, the lean table schedule (peak ~148 GB)."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


GOLD = os.path.join(os.path.dirname(__file__), "golden", "c4r_tables.json")


def c4r_norms(lat):
    """The C4r norm table for the oracle: the device walk's table, admitted
    only if it hashes to the ORACLE's own shell walk (tests/golden/
    make_c4r_golden.py, committed sha256) -- so the oracle's input is the
    oracle's index map, not the product's."""
    norm2, mx = L.aaset_norms_device(lat)
    gold = json.load(open(GOLD))
    gen, moduli = lat.generators()
    assert [int(x) for x in gen[0]] == gold["z"] and int(moduli[0]) == gold["n"]
    assert hashlib.sha256(np.ascontiguousarray(norm2, np.uint32).tobytes()).hexdigest() == gold["norm2_sha256"]
    assert int(mx) == gold["max_norm2"]
    return norm2


def test_config4_reduced_vs_oracle():
    cfg = configs.CONFIGS["C4r"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    norm2 = c4r_norms(lat)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, cfg.eps, a, b)
    orc.set_dt(cfg.dt)
    S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, norm2=norm2)
    S.set_dt(cfg.dt)
    S.discretize_initial()
    info = S.info()
    assert info["M2a"] > 0  # three-level
    g = orc.initial_samples(c[0], p[0], cfg.sigma)
    assert rel(S.get_state(L.SAMPLES)[0], g) <= 1e-13
    u0 = orc.analyze(g)
    u1 = orc.steps(u0, 1)
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= 1e-12
    u3 = orc.steps(u1, 2)
    S.step(2)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u3) <= 1e-10
    assert abs(S.l2_norm()[0] - 1.0) <= 1e-12


def test_config4_full_invariants():
    cfg = configs.CONFIGS["C4"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma)  # norm table built on the device
    S.set_dt(cfg.dt)
    S.discretize_initial()
    info = S.info()
    assert info["M2a"] > 0 and info["M"] >= 2 * cfg.N - 1
    n0 = S.l2_norm()[0]
    assert abs(n0 - 1.0) <= 1e-12
    S.step(cfg.m)
    assert abs(S.l2_norm()[0] - 1.0) <= 1e-12
    S.set_dt(-cfg.dt)
    S.step(cfg.m)
    assert S.l2_distance_initial() <= 1e-10


@pytest.mark.parametrize("world", [2, 4])
def test_config4_reduced_sharded_virtual_ranks(world):
    """Config 4's multi-GPU form: one wave function sharded
    over `world` ranks with the three-level row side (M2 = Ma x Mb inside the
    row slabs, two block exchanges per step), run as virtual ranks on one GPU
    at C4r's N, against the oracle and the unsharded solver."""
    cfg = configs.CONFIGS["C4r"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    norm2 = c4r_norms(lat)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, cfg.eps, a, b)
    orc.set_dt(cfg.dt)
    D = L.DistSolver(lat, cfg.eps, a, b, c, p, cfg.sigma, world=world, rank=-1)  # norms built on the device
    info = D.info()
    assert info["Ma"] > 0 and info["M"] >= 2 * cfg.N - 1
    assert info["M1"] % world == 0 and info["Ma"] % world == 0
    D.set_dt(cfg.dt)
    D.discretize_initial()
    g = orc.initial_samples(c[0], p[0], cfg.sigma)
    assert rel(D.get_state(), g) <= 1e-13
    assert abs(D.l2_norm() - 1.0) <= 1e-12
    u1 = orc.steps(orc.analyze(g), 1)
    D.step(1)
    assert rel(orc.analyze(D.get_state()), u1) <= 1e-12
    u3 = orc.steps(u1, 2)
    D.step(2)
    assert rel(orc.analyze(D.get_state()), u3) <= 1e-10
    assert abs(D.l2_norm() - 1.0) <= 1e-12
    # time reversibility through the sharded path
    D.set_dt(-cfg.dt)
    D.step(3)
    assert rel(D.get_state(), g) <= 1e-10
