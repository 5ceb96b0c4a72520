"""The CPU oracle pinned against SPEC.md's known answers (no GPU).

The reference has no solver, so the oracle's spectral/tdse
restatement is pinned by SPEC.md's acceptance criteria: naive-DFT equality
(crit. 1), interpolation exactness (2), aliasing identity (4), dense
matrix-exponential Strang step (5), second-order convergence (6),
commuting-case exactness (8), plus unitarity, norm conservation and
time-reversibility.
"""
import numpy as np
import pytest
import scipy.linalg

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle import pyoracle as O


@pytest.mark.parametrize("n", [1, 2, 3, 7, 55, 97, 128, 1000, 4099, 8640, 65537])
def test_fft_vs_numpy(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    X = np.fft.fft(x)
    assert np.abs(O.dft(x, -1) - X).max() <= 1e-14 * np.abs(X).max() * max(1, np.log2(n))
    assert np.abs(O.dft(x, +1) - np.fft.ifft(x) * n).max() <= 1e-14 * np.abs(X).max() * max(1, np.log2(n))


def lattice_case(kind):
    if kind == "fig1":
        return L.Lattice.rank1([1, 34], 55)
    if kind == "d3":
        z, _ = L.cbc_construct(1024, 3)
        return L.Lattice.rank1(z, 1024)
    return L.Lattice.grid([16, 16])


def oracle_for(lat, eps=0.5, a=None, b=None):
    gen, moduli = lat.generators()
    d = lat.dim()
    norm2, h, _ = L.aaset_build(lat)
    a = np.ones(d) if a is None else a
    b = np.full(max(d - 1, 1), 0.25) if b is None else b
    return O.Oracle(gen, moduli, norm2, eps, a, b), norm2, h


@pytest.mark.parametrize("kind", ["fig1", "d3", "grid"])
def test_analyze_equals_naive_dft(kind):
    # acceptance 1: 20 random fields, max rel err <= 1e-11
    lat = lattice_case(kind)
    orc, _, h = oracle_for(lat)
    p = lat.point_coords()
    E = np.exp(-2j * np.pi * (h.astype(np.float64) @ p.T))  # [chi, kappa]
    rng = np.random.default_rng(1)
    for _ in range(20):
        u = rng.standard_normal(lat.n_total()) + 1j * rng.standard_normal(lat.n_total())
        want = E @ u / lat.n_total()
        got = orc.analyze(u)
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
        assert np.abs(orc.synthesize(got) - u).max() <= 1e-12 * np.abs(u).max()
        # unitarity of sqrt(n) * analyze
        assert abs(np.linalg.norm(got) * np.sqrt(lat.n_total()) / np.linalg.norm(u) - 1) <= 1e-12


def test_interpolation_exactness():
    # acceptance 2: trig polynomial supported on A, n = 2^10, d = 3
    lat = lattice_case("d3")
    orc, _, h = oracle_for(lat)
    rng = np.random.default_rng(2)
    c = rng.standard_normal(lat.n_total()) + 1j * rng.standard_normal(lat.n_total())
    u = np.exp(2j * np.pi * (lat.point_coords() @ h.T.astype(np.float64))) @ c
    assert np.abs(orc.analyze(u) - c).max() <= 1e-10
    assert np.abs(orc.synthesize(c) - u).max() <= 1e-10 * np.abs(u).max()


def test_aliasing_identity():
    # acceptance 4: h and h + l (l dual) alias onto one coefficient
    lat = L.Lattice.rank1([1, 34], 55)
    orc, _, h = oracle_for(lat)
    ell = np.array([21, 1])  # 21 + 34 = 55: dual
    assert lat.in_dual(ell)
    p = lat.point_coords()
    hv = h[7].astype(np.float64)
    u = np.exp(2j * np.pi * p @ hv) + 2.0 * np.exp(2j * np.pi * p @ (hv + ell))
    uh = orc.analyze(u)
    want = np.zeros(55, complex)
    want[7] = 3.0
    assert np.abs(uh - want).max() <= 1e-12


def test_strang_step_dense_expm():
    # acceptance 5: d=1, n=8, one step vs the dense product
    lat = L.Lattice.rank1([1], 8)
    eps, dt = 0.7, 0.3
    a, b = np.array([1.3]), np.array([0.0])
    orc, norm2, h = oracle_for(lat, eps, a, b)
    orc.set_dt(dt)
    n = 8
    x = lat.point_coords()[:, 0]
    v = orc.potential()
    assert np.allclose(v, a[0] * (1 - np.cos(2 * np.pi * x)))
    k = np.arange(n)
    F = np.exp(-2j * np.pi * np.outer(k, k) / n) / np.sqrt(n)  # unitary F_n
    W = F @ np.diag(v) @ F.conj().T
    D = np.diag(4 * np.pi ** 2 * norm2.astype(float))
    Sw = scipy.linalg.expm(-1j / (2 * eps) * W * dt)
    Sd = scipy.linalg.expm(-1j * eps / 2 * D * dt)
    rng = np.random.default_rng(5)
    u0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert np.abs(orc.steps(u0, 1) - Sw @ Sd @ Sw @ u0).max() <= 1e-10 * np.abs(u0).max()


def test_commuting_case_exact():
    # acceptance 8: v constant -> splitting exact
    lat = L.Lattice.rank1([1, 34], 55)
    eps = 0.5
    orc, norm2, _ = oracle_for(lat, eps, np.zeros(2), np.zeros(1))
    rng = np.random.default_rng(4)
    u0 = rng.standard_normal(55) + 1j * rng.standard_normal(55)
    for dt in (0.5, 0.1):
        orc.set_dt(dt)
        m = int(round(1.0 / dt))
        exact = u0 * np.exp(-1j * eps * 1.0 * 2 * np.pi ** 2 * norm2.astype(float))
        assert np.abs(orc.steps(u0, m) - exact).max() <= 1e-10


def test_norm_reversibility_energy():
    lat, a, b, c, p = configs.small_rank1(3, 1021, seed=9)
    orc, norm2, _ = oracle_for(lat, 0.2, a, b)
    orc.set_dt(0.01)
    u0 = orc.analyze(orc.initial_samples(c[0], p[0], 0.12))
    assert abs(orc.l2_norm(u0) - 1) <= 1e-13
    u1 = orc.steps(u0, 100)
    assert abs(orc.l2_norm(u1) - orc.l2_norm(u0)) <= 1e-12
    e0, e1 = orc.energy(u0), orc.energy(u1)
    assert abs(e1 - e0) <= 1e-3 * abs(e0)
    orc.set_dt(-0.01)
    assert np.abs(orc.steps(u1, 100) - u0).max() <= 1e-10


def test_second_order_convergence():
    # acceptance 6, scaled: d=2, eps=1, seeded g and v
    lat, a, b, c, p = configs.small_rank1(2, 4099, seed=21)
    orc, _, _ = oracle_for(lat, 1.0, a, b)
    u0 = orc.analyze(orc.initial_samples(c[0], p[0], 0.12))
    T = 1.0
    orc.set_dt(T / 1024)
    ref = orc.steps(u0, 1024)
    dts, errs = [], []
    for m in (8, 16, 32, 64):
        orc.set_dt(T / m)
        errs.append(np.linalg.norm(orc.steps(u0, m) - ref))
        dts.append(T / m)
    slope = np.polyfit(np.log(dts), np.log(errs), 1)[0]
    assert 1.85 <= slope <= 2.15, (slope, errs)
