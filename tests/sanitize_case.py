"""Small propagations for compute-sanitizer (racecheck / synccheck /
memcheck), one tool per run (B200_PROFILING.md: several tools in one call
have left a GPU unusable):

    compute-sanitizer --tool racecheck --error-exitcode 9 python tests/sanitize_case.py

Covers the fused pass kernels' single-barrier ping-pong stages (the generic
fft_pass.cuh kernels and the lean per-step fft_pass4.cuh kernels, which the
solver picks for the plain layouts; LATTDSE_PASS4=0 runs the same cases on
the generic kernels only) on every program: C0 two-level circulant and the
literal Bluestein method, a three-level forced geometry, a rank-2 grid, an
ensemble with a ragged last group, and the fused observables (propagate).
Exits 0 with the solver results checked for finiteness and unit norm.
"""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1808_06357_b200 as L  # noqa: E402
from paper_1808_06357_b200 import configs  # noqa: E402


def run(S, steps):
    S.set_dt(1.0 / 64)
    S.discretize_initial()
    S.step(steps)
    n = S.l2_norm()
    assert np.all(np.abs(n - 1.0) < 1e-12), n
    return S


def main():
    cfg = configs.CONFIGS["C0"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    for method in ("circulant", "bluestein"):
        run(L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, method=method), 3)
    S = run(L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma), 1)
    S.propagate(4, 2)
    small, a2, b2, c2, p2 = configs.small_rank1(2, 4099, seed=31)
    run(L.Solver(small, 0.1, a2, b2, c2[:1], p2[:1], 0.1, geometry=(16, 24, 27)), 2)
    g2 = configs.rank2_product(64, 32, 4)
    a3, b3, c3, p3 = L.problem_draw(5, 4, 1, 0.4, 0.6, 2)
    norm2, _, _ = L.aaset_build(g2, with_vectors=False)
    run(L.Solver(g2, 0.1, a3, b3, c3, p3, 0.1, norm2=norm2), 2)
    # a two-level view whose ROW and COL lengths both run the lean pass4
    # kernels (odd first / last radices, whole tiles): 4099 points in a
    # 324 x 324 view, three members in ragged groups of two
    os.environ["LATTDSE_GEOM"] = "324x324"
    a5, b5, c5, p5 = L.problem_draw(cfg.seed, cfg.d, 3, 0.4, 0.6, 2)
    S5 = run(L.Solver(lat, cfg.eps, a5, b5, c5, p5, cfg.sigma, group=2), 2)
    assert S5.info()["pass4"] == 1 or os.environ.get("LATTDSE_PASS4") == "0", S5.info()
    del os.environ["LATTDSE_GEOM"]
    if "--quick" not in sys.argv:
        c3cfg = configs.CONFIGS["C3"]
        lat3 = configs.lattice(c3cfg)
        a4, b4, c4, p4 = configs.problem(c3cfg, batch=3)
        run(L.Solver(lat3, c3cfg.eps, a4, b4, c4, p4, c3cfg.sigma, group=2), 1)
    print("sanitize_case: ok")


if __name__ == "__main__":
    main()
