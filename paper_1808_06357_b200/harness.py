"""Experiment harness on the GPU solver: the paper's
§3.2-3.3 studies -- time-step convergence and norm / energy conservation --
re-run through the product's Solver, with the reference CLI's output
conventions: CSV series and a JSON summary carrying the
lattice hash, a config echo and the tool version.

  run_conservation  SPEC.md:479-487 -- per-record-step (step, t, norm,
                    energy, norm - norm_0, energy - energy_0); summary
                    delta_norm / delta_energy = (max - min) / mean
                    (§3.3's delta). Observables come from the
                    passes themselves (Solver.propagate: fused norm /
                    potential sums in the exit pass, kinetic sum in the
                    analysis exit pass).
  run_convergence   SPEC.md:470-477 -- l2 error of coefficient fields
                    against a fine reference run, least-squares slope of
                    log error vs log dt, points below 100 x machine epsilon
                    excluded.

    python -m paper_1808_06357_b200.harness conservation --config C1 --record-every 64 --out runs/c1
    python -m paper_1808_06357_b200.harness convergence --d 2 --n 16411 --out runs/conv
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import os
import sys

import numpy as np

from . import COEFFICIENTS, Lattice, Solver, cbc_construct, problem_draw, version

EPS_MACH = np.finfo(np.float64).eps


def _summary_base(lat: Lattice, config: dict) -> dict:
    return {"lattice_hash": f"0x{lat.hash():016x}", "lattice": json.loads(lat.to_json()), "config": config,
            "tool": version()}


def _write(out_dir, name, header, rows, summary):
    if not out_dir:
        return
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, f"{name}.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(header)
        w.writerows(rows)
    with open(os.path.join(out_dir, f"{name}.json"), "w") as f:
        json.dump(summary, f, indent=1)


def variation(x) -> float:
    """PAPER.md §3.3's delta := (max - min) / mean."""
    x = np.asarray(x, np.float64)
    if x.size == 0:
        return 0.0
    mean = float(np.mean(x))
    return float((np.max(x) - np.min(x)) / mean) if mean != 0 else float(np.max(x) - np.min(x))


def run_conservation(S: Solver, m: int, record_every: int, member: int = 0, config: dict | None = None,
                     out_dir: str | None = None) -> dict:
    """m Strang steps of `member`, observables every `record_every` steps.
    S must be set up (set_dt + discretize_initial / set_state)."""
    if m == 0:
        summary = {**_summary_base(S.lat, config or {}), "m": 0, "delta_norm": 0.0, "delta_energy": 0.0,
                   "records": 0}
        _write(out_dir, "conservation", ["step", "time", "norm", "energy", "dnorm", "denergy"], [], summary)
        return summary
    tr = S.propagate(m, record_every, member)
    norm0, en0 = tr[0, 2], tr[0, 3]
    rows = [[int(r[0]), r[1], r[2], r[3], r[2] - norm0, r[3] - en0] for r in tr]
    summary = {**_summary_base(S.lat, config or {}), "m": int(m), "record_every": int(record_every),
               "member": int(member), "dt": getattr(S, "dt", None), "records": len(rows),
               "delta_norm": variation(tr[:, 2]), "delta_energy": variation(tr[:, 3]),
               "max_abs_dnorm": float(np.max(np.abs(tr[:, 2] - norm0))),
               "max_abs_denergy": float(np.max(np.abs(tr[:, 3] - en0))), "norm0": float(norm0),
               "energy0": float(en0)}
    _write(out_dir, "conservation", ["step", "time", "norm", "energy", "dnorm", "denergy"], rows, summary)
    return summary


def fit_slope(dts, errs):
    """Least-squares slope of log err vs log dt over errors above 100 eps."""
    pts = [(math.log(d), math.log(e)) for d, e in zip(dts, errs) if e > 100 * EPS_MACH]
    if len(pts) < 2:
        return None, "exact"
    x = np.array([p[0] for p in pts])
    y = np.array([p[1] for p in pts])
    return float(np.polyfit(x, y, 1)[0]), "fit"


def run_convergence(make_solver, T: float, ms, M_ref: int, config: dict | None = None, out_dir: str | None = None,
                    member: int = 0) -> dict:
    """make_solver() -> a fresh Solver (same lattice / problem). Reference:
    M_ref steps of dt = T/M_ref; each coarse run m steps of T/m; error =
    l2 distance of the coefficient fields."""
    ms = sorted(set(int(m) for m in ms))
    if M_ref < 4 * max(ms):
        raise ValueError("reference M must exceed max(m) by a factor >= 4 (SPEC.md:464)")
    ref = make_solver()
    ref.set_dt(T / M_ref)
    ref.discretize_initial()
    ref.step(M_ref)
    uref = ref.get_state(COEFFICIENTS, m0=member, count=1)[0]
    lat = ref.lat
    del ref
    rows = []
    for m in sorted(ms):
        S = make_solver()
        S.set_dt(T / m)
        S.discretize_initial()
        S.step(m)
        err = S.l2_distance(uref, COEFFICIENTS, member)
        rows.append([T / m, err])
        del S
    slope, how = fit_slope([r[0] for r in rows], [r[1] for r in rows])
    summary = {**_summary_base(lat, config or {}), "M_ref": int(M_ref), "dt": [r[0] for r in rows],
               "l2_error": [r[1] for r in rows], "slope": slope, "slope_kind": how}
    _write(out_dir, "convergence", ["dt", "l2_error"], rows, summary)
    return summary


def _cli(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1808_06357_b200.harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("conservation", help="norm / energy conservation trace (SPEC.md:479-487)")
    c.add_argument("--config", default=None, help="BASELINE config (C0..C3); else --d/--n/--eps/--T/--m")
    c.add_argument("--d", type=int, default=5)
    c.add_argument("--n", type=int, default=1 << 16)
    c.add_argument("--eps", type=float, default=0.5)
    c.add_argument("--T", type=float, default=1.0)
    c.add_argument("--m", type=int, default=100)
    c.add_argument("--sigma", type=float, default=0.1)
    c.add_argument("--seed", type=int, default=7)
    c.add_argument("--record-every", type=int, default=1)
    c.add_argument("--member", type=int, default=0)
    c.add_argument("--out", default=None)
    v = sub.add_parser("convergence", help="time-step convergence study (SPEC.md:470-477)")
    v.add_argument("--d", type=int, default=2)
    v.add_argument("--n", type=int, default=16411)
    v.add_argument("--eps", type=float, default=1.0)
    v.add_argument("--T", type=float, default=1.0)
    v.add_argument("--ms", default="8,16,32,64,128,256")
    v.add_argument("--M-ref", type=int, default=4096)
    v.add_argument("--sigma", type=float, default=0.1)
    v.add_argument("--seed", type=int, default=7)
    v.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    if a.cmd == "conservation":
        if a.config:
            from . import configs

            cfg = configs.CONFIGS[a.config]
            lat = configs.lattice(cfg)
            pa, pb, pc, pp = configs.problem(cfg, batch=1 if cfg.batch == 1 else cfg.batch)
            S = Solver(lat, cfg.eps, pa, pb, pc, pp, cfg.sigma)
            S.set_dt(cfg.dt)
            m, echo = cfg.m, {"config": cfg.name, "d": cfg.d, "N": cfg.N, "eps": cfg.eps, "T": cfg.T, "m": cfg.m}
        else:
            z, _ = cbc_construct(a.n, a.d)
            lat = Lattice.rank1(z, a.n)
            pa, pb, pc, pp = problem_draw(a.seed, a.d, 1, 0.4, 0.6, 2)
            S = Solver(lat, a.eps, pa, pb, pc, pp, a.sigma)
            S.set_dt(a.T / a.m)
            m, echo = a.m, {"d": a.d, "n": a.n, "eps": a.eps, "T": a.T, "m": a.m, "sigma": a.sigma, "seed": a.seed}
        S.discretize_initial()
        out = run_conservation(S, m, a.record_every, a.member, echo, a.out)
    else:
        z, _ = cbc_construct(a.n, a.d)
        lat = Lattice.rank1(z, a.n)
        pa, pb, pc, pp = problem_draw(a.seed, a.d, 1, 0.4, 0.6, 2)

        def make():
            return Solver(lat, a.eps, pa, pb, pc, pp, a.sigma)

        out = run_convergence(make, a.T, [int(x) for x in a.ms.split(",")], a.M_ref,
                              {"d": a.d, "n": a.n, "eps": a.eps, "T": a.T, "sigma": a.sigma, "seed": a.seed}, a.out)
    print(json.dumps({k: out[k] for k in out if k not in ("lattice",)}))
    return 0


if __name__ == "__main__":
    sys.exit(_cli())
