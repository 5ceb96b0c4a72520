"""Device-solver harness: checkpoint/resume through
snapshots, the norm-drift watchdog of propagate, and the experiment that is
the paper's actual result -- second-order time convergence of the Strang
step (acceptance 6: slope in [1.85, 2.15]) -- re-run on the
GPU solver, at the oracle test's size and at config-1 size."""
import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs

pytestmark = pytest.mark.gpu


def _solver(lat, eps, a, b, c, p, sigma, dt):
    S = L.Solver(lat, eps, a, b, c, p, sigma)
    S.set_dt(dt)
    S.discretize_initial()
    return S


def test_resume_from_snapshot(tmp_path):
    cfg = configs.CONFIGS["C0"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    S.step(64)
    straight = S.get_state()
    S2 = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    S2.step(32)
    path = str(tmp_path / "c0.c128")
    S2.save(path, step=32, time=32 * cfg.dt)
    S2.close()
    S3 = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    meta = S3.load(path)
    assert meta["step"] == 32 and meta["dt"] == cfg.dt
    S3.step(32)
    # not bit-exact: between steps the device carries V^(1/2)-shifted samples
    # (half-step fusion), so get_state/set_state round through one extra
    # phase multiply each
    got = S3.get_state()
    assert np.linalg.norm(got - straight) <= 1e-14 * np.linalg.norm(straight)


def test_watchdog_raises_numerical_invariant():
    cfg = configs.CONFIGS["C0"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    rows = S.propagate(64, 16)  # default tolerance 1e-9: passes
    assert np.abs(rows[:, 2] - rows[0, 2]).max() <= 1e-12
    # rounding alone moves the norm by ~1e-16 per step: a 1e-300 tolerance trips
    S.set_watchdog(1e-300)
    with pytest.raises(L.LattdseError) as e:
        S.propagate(64, 16)
    assert e.value.name == "numerical_invariant"
    S.set_watchdog(0.0)  # off
    S.propagate(16, 16)


def _slope(lat, eps, a, b, c, p, sigma, T, ms, m_ref):
    S = _solver(lat, eps, a, b, c, p, sigma, T / m_ref)
    S.step(m_ref)
    ref = S.get_state(L.COEFFICIENTS)[0]
    dts, errs = [], []
    for m in ms:
        S.set_dt(T / m)
        S.discretize_initial()
        S.step(m)
        errs.append(np.linalg.norm(S.get_state(L.COEFFICIENTS)[0] - ref))
        dts.append(T / m)
    return np.polyfit(np.log(dts), np.log(errs), 1)[0], errs


def test_second_order_convergence_small():
    lat, a, b, c, p = configs.small_rank1(2, 4099, seed=21)
    slope, errs = _slope(lat, 1.0, a, b, c[:1], p[:1], 0.12, 1.0, (8, 16, 32, 64), 1024)
    assert 1.85 <= slope <= 2.15, (slope, errs)


def test_second_order_convergence_config1():
    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    # config-1 lattice, potential and initial state; eps = 1 so the
    # asymptotic regime is reached at modest m (the semiclassical eps = 0.05
    # needs dt << eps before the order shows)
    slope, errs = _slope(lat, 1.0, a, b, c, p, cfg.sigma, 0.1, (16, 32, 64, 128), 2048)
    assert 1.85 <= slope <= 2.15, (slope, errs)


# ---------------------------------------------------------------------------
# fused observables and the conservation study (§8(f) 4)
def test_fused_observables_match_oracle():
    """propagate's rows come from the fused exit-pass sums; they must equal
    the CPU oracle's norm and energy at every record."""
    from oracle.pyoracle import Oracle

    cfg = configs.CONFIGS["C0"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, norm2=norm2)
    S.set_dt(cfg.dt)
    S.discretize_initial()
    rows = S.propagate(64, 16)
    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, cfg.eps, a, b)
    orc.set_dt(cfg.dt)
    u = orc.analyze(orc.initial_samples(c[0], p[0], cfg.sigma))
    for i, r in enumerate(rows):
        if i:
            u = orc.steps(u, 16)
        assert int(r[0]) == 16 * i
        assert abs(r[2] - orc.l2_norm(u)) <= 1e-12
        e = orc.energy(u)
        assert abs(r[3] - e) <= 1e-10 * abs(e), (i, r[3], e)


def test_fused_observables_ensemble_member():
    """The fused sums are per member: a propagate of member k reports that
    member's norm and energy (checked against the unfused reductions)."""
    cfg = configs.CONFIGS["C3"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=8)
    S = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    rows = S.propagate(8, 4, member=5)
    assert abs(rows[-1, 2] - S.l2_norm()[5]) <= 1e-13
    assert abs(rows[-1, 3] - S.energy()[5]) <= 1e-11 * abs(rows[-1, 3])
    with pytest.raises(L.LattdseError) as e:
        S.propagate(4, 4, member=8)
    assert e.value.name == "invalid_argument"


def _oracle_trajectory(z, n, eps, a, b, c, p, sigma, m, stride):
    from oracle.pyoracle import Oracle, aaset

    norm2, _ = aaset([list(map(int, z))], [n], with_vectors=False)
    orc = Oracle([list(map(int, z))], [n], norm2, eps, a, b)
    orc.set_dt(1.0 / m)
    u = orc.analyze(orc.initial_samples(c, p, sigma))
    nrm, en = [orc.l2_norm(u)], [orc.energy(u)]
    for _ in range(m // stride):
        u = orc.steps(u, stride)
        nrm.append(orc.l2_norm(u))
        en.append(orc.energy(u))
    return np.array(nrm), np.array(en)


def test_conservation_acceptance7_spec_scale(tmp_path):
    """The conservation study at acceptance 7's scale: d=5,
    eps=0.5, n=2^16, dt=1/100, T=1, a record every step (the BASELINE
    seeded families stand in for g1/v2).

    delta_norm <= 1e-10 holds (unitary steps). SPEC's delta_energy <= 1e-8
    does not hold for the Strang scheme at dt = 1/100: the energy of a
    splitting method oscillates at O(dt^2) around a conserved modified
    energy, and the CPU oracle shows the same 8.2e-4 (and 2.0e-4, 5.1e-5 at
    dt = 1/200, 1/400). So the test pins the GPU trajectory to the
    oracle's record by record (norm 1e-12, energy 1e-10 relative) and
    checks the second-order scaling of delta_energy instead."""
    from paper_1808_06357_b200 import harness

    n = 1 << 16
    z, _ = L.cbc_construct(n, 5)
    lat = L.Lattice.rank1(z, n)
    a, b, c, p = L.problem_draw(7, 5, 1, 0.4, 0.6, 2)
    deltas = []
    for m in (100, 200):
        S = _solver(lat, 0.5, a, b, c, p, 0.1, 1.0 / m)
        s = harness.run_conservation(S, m, m // 100, config={"d": 5, "n": n, "eps": 0.5, "m": m},
                                     out_dir=str(tmp_path / f"m{m}"))
        assert s["records"] == 101
        assert s["delta_norm"] <= 1e-10, s["delta_norm"]
        tr = np.loadtxt(tmp_path / f"m{m}" / "conservation.csv", delimiter=",", skiprows=1)
        onrm, oen = _oracle_trajectory(z, n, 0.5, a, b, c[0], p[0], 0.1, m, m // 100)
        assert np.max(np.abs(tr[:, 2] - onrm)) <= 1e-12
        assert np.max(np.abs(tr[:, 3] - oen) / np.abs(oen)) <= 1e-10
        assert abs(s["delta_energy"] - harness.variation(oen)) <= 1e-6 * harness.variation(oen)
        deltas.append(s["delta_energy"])
    assert 3.6 <= deltas[0] / deltas[1] <= 4.4, deltas  # O(dt^2)


def test_conservation_config1_scale(tmp_path):
    """The conservation study at config-1 scale (N = 1048583, d = 6,
    eps = 0.05, 1024 steps, a record every 64 steps): norm conserved to
    1e-10 (relative variation), the final energy equal to the oracle's
    full-run fixture (tests/golden/run_C1.npz) to 1e-10 relative."""
    import os

    from paper_1808_06357_b200 import harness

    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    s = harness.run_conservation(S, cfg.m, 64, config={"config": "C1"}, out_dir=str(tmp_path))
    assert s["records"] == cfg.m // 64 + 1
    assert s["delta_norm"] <= 1e-10, s["delta_norm"]
    tr = np.loadtxt(tmp_path / "conservation.csv", delimiter=",", skiprows=1)
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "run_C1.npz"))
    e_ref = float(fx["enm_0"])
    assert abs(tr[-1, 3] - e_ref) <= 1e-10 * abs(e_ref)
    assert s["delta_energy"] <= 1e-5, s["delta_energy"]  # O(dt^2) oscillation, dt = 1/1024


def test_propagate_overhead_config1():
    """Observables at record steps cost little over plain stepping. Worst case
    of the configs: C1 (one small wave function, 57 us per step), 1024 steps,
    a record every 64. A record is the exit + re-entry pass (fused sums of
    |u|^2 and v |u|^2) and one Bluestein analysis (three passes, fused
    kinetic sum): ~5.5 steps' worth, i.e. ~9% here (measured 63.2 vs 58.1 ms,
    scripts/prop_time.py); records are asynchronous (pinned host ring, the
    host finishes record r-1 under record r's steps), a single record costs
    under 1%, and an ensemble member's record vanishes next to the step of
    all members."""
    import time

    cfg = configs.CONFIGS["C1"]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg)
    S = _solver(lat, cfg.eps, a, b, c, p, cfg.sigma, cfg.dt)
    S.step(cfg.m)  # warm the graphs
    S.propagate(128, 64)

    def best(f):
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    t_step = best(lambda: S.step(cfg.m))
    t_prop = best(lambda: S.propagate(cfg.m, 64))
    t_one = best(lambda: S.propagate(cfg.m, cfg.m))
    assert t_prop <= 1.12 * t_step, (t_prop, t_step)
    assert t_one <= 1.02 * t_step, (t_one, t_step)
