"""The lean per-step kernels (fft_pass4.cuh) against the generic pass kernels
(fft_pass.cuh) and against themselves.

compute-sanitizer is closed on this GPU pool (tests/test_gpu_sanitizer.py),
so the single-barrier ping-pong / in-place stage schemes are checked here the
way a race would show: (1) the two kernel families, which share no stage
code, agree to rounding on every layout pass4 serves; (2) repeated runs of
the same propagation are bit-identical although CTA scheduling differs from
run to run; (3) results do not depend on how many members share a launch.
"""
import os

import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs

pytestmark = pytest.mark.gpu


def _solver(lat, eps, a, b, c, p, sigma, dt, pass4=True, geom=None, norm2=None, **kw):
    old = {k: os.environ.get(k) for k in ("LATTDSE_PASS4", "LATTDSE_GEOM")}
    try:
        os.environ["LATTDSE_PASS4"] = "1" if pass4 else "0"
        if geom:
            os.environ["LATTDSE_GEOM"] = geom
        S = L.Solver(lat, eps, a, b, c, p, sigma, norm2=norm2, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    S.set_dt(dt)
    S.discretize_initial()
    return S


def _rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@pytest.mark.parametrize("geom", ["486x1080", "1080x486", "324x1620", "729x720", "810x648"])
def test_pass4_matches_generic_kernels_config3_shapes(geom):
    cfg = configs.CONFIGS["C3"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=8)
    S4 = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, pass4=True, geom=geom)
    S1 = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, pass4=False, geom=geom)
    S4.step(5)
    S1.step(5)
    assert S4.info()["pass4"] == 1 and S1.info()["pass4"] == 0
    assert (S4.info()["M1"], S4.info()["M2"]) == tuple(int(x) for x in geom.split("x"))
    g4, g1 = S4.get_state(L.SAMPLES), S1.get_state(L.SAMPLES)
    for m in range(8):
        assert _rel(g4[m], g1[m]) <= 2e-14, (geom, m)
    assert np.all(np.abs(S4.l2_norm() - 1.0) <= 1e-12)


def test_pass4_config1_and_rank2():
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S4 = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, pass4=True)
    S1 = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt, pass4=False)
    S4.step(16)
    S1.step(16)
    assert S4.info()["pass4"] == 1
    assert _rel(S4.get_state(L.SAMPLES)[0], S1.get_state(L.SAMPLES)[0]) <= 5e-14
    # rank-2 grid with odd-radix sides: the LUT-diagonal COL variant and the plain ROW variant
    g2 = configs.rank2_product(324, 324, 4)
    a3, b3, c3, p3 = L.problem_draw(5, 4, 2, 0.4, 0.6, 2)
    norm2, _, _ = L.aaset_build(g2, with_vectors=False)
    R4 = _solver(g2, 0.1, a3, b3, c3, p3, 0.1, 1.0 / 64, pass4=True, norm2=norm2)
    R1 = _solver(g2, 0.1, a3, b3, c3, p3, 0.1, 1.0 / 64, pass4=False, norm2=norm2)
    R4.step(4)
    R1.step(4)
    assert R4.info()["pass4"] == 1
    r4, r1 = R4.get_state(L.SAMPLES), R1.get_state(L.SAMPLES)
    for m in range(2):
        assert _rel(r4[m], r1[m]) <= 2e-14


def test_pass4_repeated_runs_bit_identical_and_batch_independent():
    cfg = configs.CONFIGS["C3"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=24)
    outs = []
    for _ in range(3):
        S = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
        S.step(12)
        outs.append(S.get_state(L.SAMPLES).copy())
    assert np.array_equal(outs[0].view(np.uint64), outs[1].view(np.uint64))
    assert np.array_equal(outs[0].view(np.uint64), outs[2].view(np.uint64))
    # the same members alone (another grid shape, other co-resident CTAs): identical bits
    S = _solver(lat, cfg.eps, a, b, c[5:8], p[5:8], cfg.sigma, cfg.dt)
    S.step(12)
    assert np.array_equal(S.get_state(L.SAMPLES).view(np.uint64), outs[0][5:8].view(np.uint64))
