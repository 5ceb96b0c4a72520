"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle.

Tolerances (BASELINE.json north_star): relative L2 difference of the wave
function <= 1e-12 after one step and <= 1e-10 after the full run;
| ||u|| - 1 | <= 1e-12 (norm conservation). Index maps / generating vectors are
compared bit-exactly in the CPU tests.
"""
import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle.pyoracle import Oracle

pytestmark = pytest.mark.gpu

TOL_ONE = 1e-12
TOL_RUN = 1e-10
TOL_NORM = 1e-12


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def make(lat, a, b, c, p, sigma, eps, dt, method="circulant", batch=None):
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, eps, a, b)
    orc.set_dt(dt)
    S = L.Solver(lat, eps, a, b, c if batch is None else c[:batch], p if batch is None else p[:batch], sigma,
                 method=method, norm2=norm2)
    S.set_dt(dt)
    S.discretize_initial()
    return S, orc


def oracle_coeffs(orc, c, p, sigma, steps):
    g = orc.initial_samples(c, p, sigma)
    u0 = orc.analyze(g)
    return g, u0, orc.steps(u0, steps)


@pytest.mark.parametrize("method", ["circulant", "bluestein"])
@pytest.mark.parametrize("n,d", [(5, 1), (8, 1), (55, 2), (101, 3), (4099, 2), (16411, 4)])
def test_rank1_small(n, d, method):
    lat, a, b, c, p = configs.small_rank1(d, n, seed=11 + n)
    eps, dt, sigma = 0.1, 1.0 / 64, 0.12
    S, orc = make(lat, a, b, c, p, sigma, eps, dt, method)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], sigma, 1)
    # discretisation matches the oracle's samples and coefficients
    assert rel(S.get_state(L.SAMPLES)[0], g) <= 1e-14
    assert rel(S.get_state(L.COEFFICIENTS)[0], u0) <= 1e-13
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    u10 = orc.steps(u1, 9)
    S.step(9)
    got = S.get_state(L.COEFFICIENTS)[0]
    assert rel(got, u10) <= TOL_RUN
    assert abs(S.l2_norm()[0] - orc.l2_norm(u10)) <= TOL_NORM
    assert abs(S.energy()[0] - orc.energy(u10)) <= 1e-10 * abs(orc.energy(u10))


def test_config0_full_run():
    cfg = configs.CONFIGS["C0"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S, orc = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], cfg.sigma, 1)
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    um = orc.steps(u1, cfg.m - 1)
    S.step(cfg.m - 1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], um) <= TOL_RUN
    assert abs(S.l2_norm()[0] - 1.0) <= TOL_NORM


def test_config0_bluestein_matches_circulant():
    cfg = configs.CONFIGS["C0"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S1, _ = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt, "circulant")
    S2, _ = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt, "bluestein")
    S1.step(cfg.m)
    S2.step(cfg.m)
    assert rel(S1.get_state()[0], S2.get_state()[0]) <= TOL_RUN


@pytest.mark.parametrize("n1,n2,d", [(4, 4, 2), (16, 16, 3), (64, 32, 4), (256, 256, 4)])
def test_rank2_grid_small(n1, n2, d):
    lat = configs.rank2_product(n1, n2, d)
    a, b, c, p = L.problem_draw(99 + n1, d, 1, 0.4, 0.6, 2)
    eps, dt, sigma = 0.05, 1.0 / 32, 0.15
    S, orc = make(lat, a, b, c, p, sigma, eps, dt)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], sigma, 1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u0) <= 1e-13
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    u8 = orc.steps(u1, 7)
    S.step(7)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u8) <= TOL_RUN


def _rank_r_lattice(kind):
    if kind == "grid3":
        return L.Lattice.grid([64, 32, 16])
    if kind == "grid4":
        return L.Lattice.grid([16, 16, 8, 8])
    if kind == "odd3":  # odd-radix sides: the lean pass4 kernels where the tiles are whole
        return L.Lattice.grid([81, 27, 9])
    # rank 3 in five dimensions: block generators (1, 19 | 1, 7 | 1) over moduli 64, 32, 16
    return L.Lattice.create(5, 3, [[1, 19, 0, 0, 0], [0, 0, 1, 7, 0], [0, 0, 0, 0, 1]], [64, 32, 16])


@pytest.mark.parametrize("kind", ["grid3", "block3", "grid4", "odd3"])
def test_rank_r_grid(kind):
    """rank-r lattices, r >= 3: the r-dim DFT
    axis by axis -- first-axis COL pass with the kinetic diagonal, plain
    passes along the axes between, last-axis ROW pass with the potential."""
    lat = _rank_r_lattice(kind)
    d = lat.dim()
    a, b, c, p = L.problem_draw(321 + d, d, 2, 0.4, 0.6, 2)
    eps, dt, sigma = 0.05, 1.0 / 32, 0.2
    S, orc = make(lat, a, b, c, p, sigma, eps, dt)
    assert S.info()["rank"] == lat.rank() >= 3
    for m in range(2):
        g, u0, u1 = oracle_coeffs(orc, c[m], p[m], sigma, 1)
        assert rel(S.get_state(L.COEFFICIENTS)[m], u0) <= 1e-13
    S.step(1)
    for m in range(2):
        g, u0, u1 = oracle_coeffs(orc, c[m], p[m], sigma, 1)
        assert rel(S.get_state(L.COEFFICIENTS)[m], u1) <= TOL_ONE
    S.step(7)
    for m in range(2):
        g, u0, u8 = oracle_coeffs(orc, c[m], p[m], sigma, 8)
        assert rel(S.get_state(L.COEFFICIENTS)[m], u8) <= TOL_RUN
    assert np.all(np.abs(S.l2_norm() - 1.0) <= 1e-12)
    e_gpu = S.energy()
    for m in range(2):
        g, u0, u8 = oracle_coeffs(orc, c[m], p[m], sigma, 8)
        assert abs(e_gpu[m] - orc.energy(u8)) <= 1e-10 * abs(orc.energy(u8))


def test_batch_members_independent():
    lat, a, b, c, p = configs.small_rank1(3, 1021, seed=5, batch=6, c_range=(0.3, 0.7), p_max=3)
    eps, dt, sigma = 0.05, 1.0 / 128, 0.1
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, eps, a, b)
    orc.set_dt(dt)
    # groups of 4 and of 1 must give identical (bit-for-bit) results
    outs = []
    for group in (4, 1):
        S = L.Solver(lat, eps, a, b, c, p, sigma, group=group, norm2=norm2)
        S.set_dt(dt)
        S.discretize_initial()
        S.step(3)
        outs.append(S.get_state())
    assert np.array_equal(outs[0], outs[1])
    for m in range(6):
        _, _, u3 = oracle_coeffs(orc, c[m], p[m], sigma, 3)
        assert rel(orc.analyze(outs[0][m]), u3) <= TOL_ONE * 10


def test_time_reversibility_and_norm():
    lat, a, b, c, p = configs.small_rank1(4, 16411, seed=3)
    eps, dt, sigma = 0.1, 1.0 / 50, 0.1
    S, _ = make(lat, a, b, c, p, sigma, eps, dt)
    u0 = S.get_state()[0]
    S.step(50)
    assert abs(S.l2_norm()[0] - 1.0) <= TOL_NORM
    S.set_dt(-dt)
    S.step(50)
    assert rel(S.get_state()[0], u0) <= 1e-10


def test_commuting_case_constant_potential():
    # v == const (a = b = 0 gives v = 0): splitting exact, u(T) = exp(-i eps T 2pi^2 |h|^2) u0
    lat, _, _, c, p = configs.small_rank1(2, 4099, seed=2)
    a = np.zeros(2)
    b = np.zeros(1)
    eps, dt, sigma = 0.1, 0.5, 0.1
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    S = L.Solver(lat, eps, a, b, c, p, sigma, norm2=norm2)
    S.set_dt(dt)
    S.discretize_initial()
    u0 = S.get_state(L.COEFFICIENTS)[0]
    S.step(2)
    exact = u0 * np.exp(-1j * eps * 1.0 * 2 * np.pi ** 2 * norm2.astype(np.float64))
    assert rel(S.get_state(L.COEFFICIENTS)[0], exact) <= 1e-10


def test_config1_first_steps():
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S, orc = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], cfg.sigma, 1)
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    u4 = orc.steps(u1, 3)
    S.step(3)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u4) <= TOL_ONE * 4


def test_config1_full_run_invariants():
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S, _ = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt)
    e0 = S.energy()[0]
    S.step(cfg.m)
    assert abs(S.l2_norm()[0] - 1.0) <= TOL_NORM
    e1 = S.energy()[0]
    assert abs(e1 - e0) <= 1e-3 * abs(e0)  # Strang energy error O(dt^2), bounded


def test_config2_first_step():
    cfg = configs.CONFIGS["C2"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S, orc = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], cfg.sigma, 1)
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    S.step(cfg.m - 1)
    assert abs(S.l2_norm()[0] - 1.0) <= TOL_NORM


@pytest.mark.parametrize("cluster", ["8", "4", "2"])
def test_config2_cluster_col_opt_in(cluster, monkeypatch):
    """Config 2 with the opt-in cluster COL pass (LATTDSE_CLUSTER_COL: each
    4096-long column split over a cluster of 8 or 4 CTAs through distributed
    shared memory, cluster_col.inl) against the oracle."""
    if "experimental" not in L.version():
        pytest.skip("cluster COL pass not in this build (make EXPERIMENTAL=1)")
    monkeypatch.setenv("LATTDSE_CLUSTER_COL", cluster)
    cfg = configs.CONFIGS["C2"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S, orc = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], cfg.sigma, 1)
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    u3 = orc.steps(u1, 2)
    S.step(2)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u3) <= TOL_RUN
    assert abs(S.l2_norm()[0] - 1.0) <= TOL_NORM


def test_config3_members_vs_oracle():
    cfg = configs.CONFIGS["C3"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    batch = 8
    S, orc = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt, batch=batch)
    S.step(2)
    got = S.get_state(L.COEFFICIENTS)
    for m in (0, 3, 7):
        _, _, u2 = oracle_coeffs(orc, c[m], p[m], cfg.sigma, 2)
        assert rel(got[m], u2) <= TOL_ONE * 2
    assert np.all(np.abs(S.l2_norm() - 1.0) <= TOL_NORM)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_virtual_ranks(world):
    """Sharded single wave function (slabs + block exchanges) on `world`
    virtual ranks of one GPU vs the unsharded solver and the oracle."""
    lat, a, b, c, p = configs.small_rank1(4, 16411, seed=17)
    eps, dt, sigma = 0.1, 1.0 / 64, 0.1
    S, orc = make(lat, a, b, c, p, sigma, eps, dt)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    D = L.DistSolver(lat, eps, a, b, c, p, sigma, world=world, rank=-1, norm2=norm2)
    D.set_dt(dt)
    D.discretize_initial()
    assert rel(D.get_state(), S.get_state()[0]) <= 1e-15
    D.step(1)
    S.step(1)
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], sigma, 1)
    assert rel(orc.analyze(D.get_state()), u1) <= TOL_ONE
    D.step(9)
    S.step(9)
    assert rel(D.get_state(), S.get_state()[0]) <= 1e-12
    assert abs(D.l2_norm() - 1.0) <= TOL_NORM
    assert D.info()["M1"] % world == 0 and D.info()["M2"] % world == 0


@pytest.mark.parametrize("world", [4, 8])
def test_sharded_config1(world):
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S, orc = make(lat, a, b, c, p, cfg.sigma, cfg.eps, cfg.dt)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    D = L.DistSolver(lat, cfg.eps, a, b, c, p, cfg.sigma, world=world, rank=-1, norm2=norm2)
    D.set_dt(cfg.dt)
    D.discretize_initial()
    D.step(4)
    S.step(4)
    assert rel(D.get_state(), S.get_state()[0]) <= 1e-12
    assert abs(D.l2_norm() - 1.0) <= TOL_NORM


def make_geom(lat, a, b, c, p, sigma, eps, dt, geometry, method="circulant"):
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, eps, a, b)
    orc.set_dt(dt)
    S = L.Solver(lat, eps, a, b, c[:1], p[:1], sigma, method=method, norm2=norm2, geometry=geometry)
    S.set_dt(dt)
    S.discretize_initial()
    return S, orc


@pytest.mark.parametrize("chunk", [0, 1, 5])
@pytest.mark.parametrize("method", ["circulant", "bluestein"])
@pytest.mark.parametrize("geom", [(16, 24, 27), (9, 32, 32), (27, 9, 48)])
def test_three_level_forced(geom, method, chunk, monkeypatch):
    """Three-level rank-1 layout (M = M1 x Ma x Mb: COL pass, then a COL pass
    inside every row and a ROW pass) forced at a small N against the oracle;
    chunk > 0 forces the L2-chunked row side (chunk rows of the M1 x M2 view
    at a time; 5 leaves a ragged last chunk), the opt-in LATTDSE_ROW_CHUNK."""
    if chunk:
        if "experimental" not in L.version():
            pytest.skip("L2 row chunks not in this build (make EXPERIMENTAL=1)")
        monkeypatch.setenv("LATTDSE_ROW_CHUNK", str(chunk))
    lat, a, b, c, p = configs.small_rank1(2, 4099, seed=31)
    eps, dt, sigma = 0.1, 1.0 / 64, 0.1
    S, orc = make_geom(lat, a, b, c, p, sigma, eps, dt, geom, method)
    info = S.info()
    assert (info["M1"], info["M2a"], info["M2"]) == (geom[0], geom[1], geom[1] * geom[2])
    assert info["row_chunk"] == chunk
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], sigma, 1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u0) <= 1e-13
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    u10 = orc.steps(u1, 9)
    S.step(9)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u10) <= TOL_RUN
    assert abs(S.l2_norm()[0] - orc.l2_norm(u10)) <= TOL_NORM


def test_three_level_automatic_beyond_two_level_range():
    """N = smallest prime >= 2^23: 2N-1 exceeds 4096 x 4096, so the solver
    must pick a three-level view on its own."""
    n = 8388617
    # z = cbc_construct(n, 3) (78 s on 8 host cores, so fixed here)
    lat = L.Lattice.rank1([1, 2480387, 663367], n)
    a, b, c, p = L.problem_draw(41, 3, 1, 0.4, 0.6, 2)
    eps, dt, sigma = 0.05, 1.0 / 128, 0.1
    S, orc = make_geom(lat, a, b, c, p, sigma, eps, dt, None)
    info = S.info()
    assert info["M2a"] > 0 and info["M"] >= 2 * n - 1
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], sigma, 1)
    S.step(1)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u1) <= TOL_ONE
    u4 = orc.steps(u1, 3)
    S.step(3)
    assert rel(S.get_state(L.COEFFICIENTS)[0], u4) <= TOL_RUN
    assert abs(S.l2_norm()[0] - 1.0) <= TOL_NORM


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_three_level_automatic(world):
    """N = 8388617: no two-level split covers 2N-1, so the sharded solver
    runs three-level rows (Ma x Mb inside the row slabs) on its own; virtual
    ranks vs the unsharded solver and the oracle."""
    n = 8388617
    lat = L.Lattice.rank1([1, 2480387, 663367], n)
    a, b, c, p = L.problem_draw(41, 3, 1, 0.4, 0.6, 2)
    eps, dt, sigma = 0.05, 1.0 / 128, 0.1
    S, orc = make_geom(lat, a, b, c, p, sigma, eps, dt, None)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    D = L.DistSolver(lat, eps, a, b, c, p, sigma, world=world, rank=-1, norm2=norm2)
    info = D.info()
    assert info["Ma"] > 0 and info["Ma"] * info["Mb"] == info["M2"]
    assert info["M1"] % world == 0 and info["Ma"] % world == 0
    D.set_dt(dt)
    D.discretize_initial()
    assert rel(D.get_state(), S.get_state()[0]) <= 1e-15
    g, u0, u1 = oracle_coeffs(orc, c[0], p[0], sigma, 1)
    D.step(1)
    assert rel(orc.analyze(D.get_state()), u1) <= TOL_ONE
    D.step(3)
    S.step(4)
    assert rel(D.get_state(), S.get_state()[0]) <= 1e-12
    assert abs(D.l2_norm() - 1.0) <= TOL_NORM
