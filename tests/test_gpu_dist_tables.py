"""DistSolver.set_dt builds its propagator tables slab by slab (solver_dist.cu):
no unsharded table solver, peak memory per rank ~ 1/G of the problem.

Virtual ranks on one GPU (the exchanges are device copies); the NCCL backend
runs the same code with one rank per process.
"""
import os

import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _dist(lat, eps, a, b, c, p, sigma, dt, world, norm2, mode=None):
    old = os.environ.get("LATTDSE_DIST_TABLES")
    try:
        if mode:
            os.environ["LATTDSE_DIST_TABLES"] = mode
        else:
            os.environ.pop("LATTDSE_DIST_TABLES", None)
        D = L.DistSolver(lat, eps, a, b, c, p, sigma, world=world, rank=-1, norm2=norm2)
        D.set_dt(dt)
    finally:
        if old is None:
            os.environ.pop("LATTDSE_DIST_TABLES", None)
        else:
            os.environ["LATTDSE_DIST_TABLES"] = old
    D.discretize_initial()
    return D


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_tables_equal_sliced_tables_config1(world):
    """Same stepping results from slab-built tables and from the sliced tables
    of an unsharded solver (the round-1 path), and against the unsharded solver."""
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    Ds = _dist(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, world, norm2)
    Df = _dist(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, world, norm2, mode="full")
    S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, norm2=norm2)
    S.set_dt(cfg.dt)
    S.discretize_initial()
    for D in (Ds, Df):
        D.step(6)
    S.step(6)
    assert rel(Ds.get_state(), Df.get_state()) <= 2e-13
    assert rel(Ds.get_state(), S.get_state()[0]) <= 1e-12
    assert abs(Ds.l2_norm() - 1.0) <= 1e-12
    # time reversal with slab-built tables for -dt
    Ds.set_dt(-cfg.dt)
    Ds.step(6)
    S2 = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, norm2=norm2)
    S2.set_dt(cfg.dt)
    S2.discretize_initial()
    assert rel(Ds.get_state(), S2.get_state()[0]) <= 1e-10


def test_sharded_tables_three_level_and_device_norms():
    """N = 8388617 takes the three-level rows; norm table built on the device
    (empty norm2), tables built on the slabs; against the unsharded solver."""
    lat, a, b, c, p = configs.small_rank1(4, 8388617, seed=3)
    eps, dt, sigma = 0.05, 1.0 / 128, 0.1
    D = _dist(lat, eps, a, b, c, p, sigma, dt, 2, None)
    assert D.info()["Ma"] > 0
    S = L.Solver(lat, eps, a, b, c, p, sigma)
    S.set_dt(dt)
    S.discretize_initial()
    D.step(3)
    S.step(3)
    assert rel(D.get_state(), S.get_state()[0]) <= 1e-12
    assert abs(D.l2_norm() - 1.0) <= 1e-12


def test_table_peak_memory_scales_with_ranks():
    """Per-rank peak of set_dt: about 7 slabs of 16 M / G bytes + 2 N bytes of
    norm index; the sliced-table path holds the whole unsharded solver."""
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    peaks = {}
    for world in (2, 4, 8):
        D = _dist(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, world, norm2)
        info = D.info()
        peaks[world] = info["table_peak_bytes"]
        slab = 16.0 * info["M"] / world
        assert peaks[world] <= 7.5 * slab + 2.0 * cfg.N + 8e6, (world, peaks[world], slab)
        del D
    assert peaks[4] <= 0.62 * peaks[2] and peaks[8] <= 0.62 * peaks[4], peaks
    Df = _dist(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, 8, norm2, mode="full")
    assert Df.info()["table_peak_bytes"] >= 3.0 * peaks[8]


@pytest.mark.parametrize("chunks", [3])
def test_chunked_overlapped_row_side_identical(chunks, monkeypatch):
    """The pipelined row side (exchange chunks on their own stream under the
    row passes of the other chunks) gives bit-identical results to the
    blocking exchanges: two-level (config 1, 4 ranks) and three-level rows."""
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    monkeypatch.delenv("LATTDSE_DIST_CHUNKS", raising=False)
    D1 = _dist(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, 4, norm2)
    monkeypatch.setenv("LATTDSE_DIST_CHUNKS", str(chunks))
    Dk = _dist(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, 4, norm2)
    D1.step(5)
    Dk.step(5)
    assert np.array_equal(D1.get_state().view(np.uint64), Dk.get_state().view(np.uint64))
    lat3, a3, b3, c3, p3 = configs.small_rank1(4, 8388617, seed=3)
    monkeypatch.delenv("LATTDSE_DIST_CHUNKS", raising=False)
    E1 = _dist(lat3, 0.05, a3, b3, c3, p3, 0.1, 1.0 / 128, 2, None)
    monkeypatch.setenv("LATTDSE_DIST_CHUNKS", str(chunks))
    Ek = _dist(lat3, 0.05, a3, b3, c3, p3, 0.1, 1.0 / 128, 2, None)
    E1.step(2)
    Ek.step(2)
    assert np.array_equal(E1.get_state().view(np.uint64), Ek.get_state().view(np.uint64))
