"""Benchmark of the Strang time-stepping hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C1] [--method circulant|bluestein]

Workload (config.workload): BASELINE.json configs[1] = C1, d=6 rank-1
lattice, N = 1048583 (smallest prime >= 2^20), eps=0.05, T=1, m=1024, one
complex fp64 wave function. One bench step = one full propagation
(m = 1024 Strang steps) of that wave function. L2 is flushed
(512 MiB memset) before every timed bench step, outside its event pair.

value    : lattice-point Strang steps/s = N * m * ranks / (max over ranks of the
           summed device time of the K steps), CUDA events on the solver stream.
e2e      : the same metric through the public API with host buffers: per step
           set_state from pinned host memory (H2D), step(m), get_state (D2H),
           wall clock around the synchronous calls.
roofline : dominant pass kernel, algorithmic bytes per launch / its average
           event-timed duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: the CPU oracle (oracle/, a port of the reference spec -- the
           reference itself has no solver) on this host's cores, bounded sample.
--impl reference: that CPU port on all host threads, same metric and config.
N > 1 (torchrun): C1 does not shard -- every rank runs an independent replica
("replicas only"); barrier + max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "lattice-point Strang steps/s (fp64 complex)"
UNIT = "lattice-pt-steps/s"


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        return world, rank, local, dist, torch
    return 1, 0, 0, None, None


def _dev(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(x, dist, torch):
    if dist is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, dist, torch):
    if dist is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ------------------------------------------------------------------ CPU port
def cpu_port_rate(cfg, lat, norm2, a, b, c, p, steps_per_sample: int, samples: int = 1):
    """CPU oracle (all threads): lattice-pt-steps/s over a bounded sample."""
    from oracle.pyoracle import Oracle

    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, cfg.eps, a, b)
    orc.set_dt(cfg.dt)
    u = orc.analyze(orc.initial_samples(c[0], p[0], cfg.sigma))
    orc.steps(u, 1)  # warm the plans
    times = []
    for _ in range(samples):
        t0 = time.perf_counter()
        u = orc.steps(u, steps_per_sample)
        times.append(time.perf_counter() - t0)
    return cfg.N * steps_per_sample / statistics.mean(times), times


CPU_MAX_N = 1 << 25  # the CPU port is timed on configs up to this size


def cpu_case(cfg):
    """(config, lattice, norm table, a, b, c, p, note) the CPU port is timed on:
    the workload itself, or -- config 4, whose single state is 17 GB and whose
    CPU step takes minutes -- its reduced-N twin C4r (same d, eps, T, m,
    sigma; N = 16777259), the rate being per lattice-point step either way."""
    import paper_1808_06357_b200 as L
    from paper_1808_06357_b200 import configs

    note = ""
    if cfg.N > CPU_MAX_N and "C4r" in configs.CONFIGS:
        cfg = configs.CONFIGS["C4r"]
        note = " (C4r: config 4's shape at N = 16777259; the full-N CPU step does not fit a bounded sample)"
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=1)
    if cfg.rank == 1 and cfg.d > 8:
        # d = 20: the host shell walk takes hours; the oracle's norm-table INPUT is
        # built on the device (bit-identical to the host walk, tests/test_gpu_setup.py)
        norm2, _ = L.aaset_norms_device(lat)
    else:
        norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    return cfg, lat, norm2, a, b, c, p, note


def run_reference(args, cfg):
    world, rank, _, dist, torch = dist_setup(args.gpus)
    if rank != 0:
        return 0
    ccfg, lat, norm2, a, b, c, p, note = cpu_case(cfg)
    sample = max(1, args.ref_sample_steps)
    for _ in range(args.warmup):
        cpu_port_rate(ccfg, lat, norm2, a, b, c, p, 1)
    rate, times = cpu_port_rate(ccfg, lat, norm2, a, b, c, p, sample, samples=args.steps)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (complex fp64)", "data": "synthetic (seeded BASELINE families)",
        "config": config_dict(cfg, args, note=f"1 reference step = {sample} Strang steps of the workload (bounded sample)"),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{sample} literal Strang steps of {ccfg.name} per bench step (4 length-N DFTs each), "
                                   f"OpenMP on {cores} host threads{note}"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg, args, note=None):
    d = {"workload": f"{cfg.name}: d={cfg.d} rank-{cfg.rank} N={cfg.N} eps={cfg.eps} T={cfg.T} m={cfg.m} "
                     f"batch={cfg.batch}; 1 bench step = full propagation (m Strang steps)",
         "lattice": "CBC prime-n generating vector (paper_1808_06357_b200/catalog.json)" if cfg.rank == 1
         else "product rank-2 lattice (configs.py)",
         "method": args.method, "l2": "flushed (512 MiB memset) before every timed bench step",
         "parallelism": ("1 GPU" if args.gpus == 1 else
                         ("ensemble sharded by member (shard_members), no data-path collective" if cfg.batch > 1
                          else "replicas only (a single wave function of this size does not shard)"))}
    if note:
        d["note"] = note
    return d


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg):
    world, rank, local, dist, torch = dist_setup(args.gpus)
    import paper_1808_06357_b200 as L
    from paper_1808_06357_b200 import configs

    lat = configs.lattice(cfg)
    batch_total = cfg.batch if args.batch is None else args.batch
    a, b, c, p = configs.problem(cfg, batch=batch_total)
    if batch_total > 1:
        # ensemble: shard members across ranks, no data-path collective
        m0, batch = configs.shard_members(batch_total, rank, world)
        c, p = c[m0:m0 + batch], p[m0:m0 + batch]
        members_all = batch_total
    else:
        batch = 1  # single wave function: every rank runs a replica
        members_all = world
    # rank-1: the solver builds its norm table on the device (setup, untimed)
    norm2 = None if cfg.rank == 1 else L.aaset_build(lat, with_vectors=False)[0]
    S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, method=args.method, device=local, norm2=norm2)
    S.set_dt(cfg.dt)
    S.discretize_initial()
    info = S.info()
    m = cfg.m if args.m is None else args.m

    for _ in range(args.warmup):
        S.step(m)

    # ---- timed region: K bench steps, each a full propagation, L2 flushed before each
    clocks = Clocks(local)
    barrier(dist)
    S.synchronize()
    clocks.start()
    launches0 = S.kernel_launches()
    per_step = []
    for _ in range(args.steps):
        S.flush_l2()
        per_step.append(S.time_steps(m))
    S.synchronize()
    launches = S.kernel_launches() - launches0
    clk = clocks.stop()
    barrier(dist)
    total_ms = max_over_ranks(sum(per_step), dist, torch)
    work = float(cfg.N) * members_all * m * args.steps
    value = work / (total_ms * 1e-3)

    # ---- per-pass durations (instrumented run, outside the timed region)
    S.flush_l2()
    ms_col, ms_row = S.profile_passes(min(m, 256))
    peak, peak_kind = measured_hbm_peak()
    dom = "col" if ms_col >= ms_row else "row"
    dom_ms = ms_col if dom == "col" else ms_row
    # info's per-pass bytes cover the whole batch; one launch covers one group
    groups = -(-batch // max(1, info["group"]))
    dom_bytes = (info["bytes_per_pass_col"] if dom == "col" else info["bytes_per_pass_row"]) / groups
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"{cfg.name}_{args.method}_{dom}")
        except Exception:
            traffic = None
    step_ms = statistics.mean(per_step) / m
    canonical = (160.0 * info["M"] + 18.0 * info["n_total"]) * batch if cfg.rank == 1 else 82.0 * info["n_total"] * batch
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "kernel": f"{dom} pass (fft_pass_kernel, {'COL' if dom == 'col' else 'ROW'} axis)",
        "bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms, "peak_kind": peak_kind,
        "pass_ms": {"col": ms_col, "row": ms_row},
        "note": (f"working set ~{info['bytes_per_step'] / 2 / 1e6:.0f} MB per pass: L2-resident across steps (126 MB L2); "
                 "frac > 1 would mean L2 reuse, see DESIGN.md" if info["bytes_per_step"] / 2 < 100e6 else
                 f"working set {info['bytes_per_step'] / 2 / 1e9:.1f} GB per pass streams through HBM"),
        "step_vs_canonical": {
            "canonical_bytes_per_step": canonical,
            "canonical_model": "160*M*+18*N (4 Bluestein passes, SURVEY.md 8(d))" if cfg.rank == 1 else "82*N",
            "t_roof_us_at_8TBps": canonical / 8e12 * 1e6, "measured_us_per_step": step_ms * 1e3,
            "frac_of_canonical_roofline": (canonical / 8e12) / (step_ms * 1e-3)},
    }

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if rank == 0 or world > 1:
        import torch as _t

        n = cfg.N * batch
        host_in = _t.empty(2 * n, dtype=_t.float64, pin_memory=True)
        host_out = _t.empty(2 * n, dtype=_t.float64, pin_memory=True)
        g = S.get_state()
        host_in.numpy()[:] = g.reshape(-1).view(np.float64)
        e2e_times = []
        for _ in range(args.steps):
            S.flush_l2()
            t0 = time.perf_counter()
            S.set_state_ptr(host_in.data_ptr(), batch)
            S.step(m)
            S.get_state_ptr(host_out.data_ptr(), batch)
            e2e_times.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(e2e_times), dist, torch)
        e2e = {"value": float(cfg.N) * members_all * m * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n,
               "ms_per_step": 1e3 * e2e_s / args.steps}

    # ---- CPU baseline (rank 0, N=1 only): oracle port, bounded sample
    cpu = None
    if world == 1 and not args.no_cpu:
        ccfg, clat, cnorm2, ca, cb, cc, cp, note = cpu_case(cfg)
        rate1, _ = cpu_port_rate(ccfg, clat, cnorm2, ca, cb, cc, cp, 1)
        steps = max(1, min(64, int(args.cpu_seconds / max(ccfg.N / rate1, 1e-3))))
        rate, times = cpu_port_rate(ccfg, clat, cnorm2, ca, cb, cc, cp, steps)
        cpu = {"value": rate, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"{steps} literal Strang steps of {ccfg.name} (CPU oracle, OpenMP on {os.cpu_count()} threads), "
                         f"{sum(times):.1f} s{note}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if batch_total > 1 else "weak", "vs_baseline": None, "dtype": "c128 (complex fp64)",
            "data": "synthetic (seeded BASELINE families, DESIGN.md Seeds)",
            "config": config_dict(cfg, args), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk,
            "solver": {k: info[k] for k in ("M", "M1", "M2", "group", "launches_per_step", "bytes_per_step")},
            "us_per_strang_step": step_ms * 1e3,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- sharded arm
def run_sharded(args, cfg):
    """One wave function sharded over the ranks (DistSolver): NCCL exchanges
    between GPUs under torchrun, or --virtual-ranks G on one GPU."""
    world, rank, local, dist, torch = dist_setup(args.gpus)
    import paper_1808_06357_b200 as L
    from paper_1808_06357_b200 import configs

    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=1)
    norm2 = None  # rank-1: the norm table is built on the device (bit-identical to the host walk)
    if world > 1:
        uid = [L.DistSolver.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        D = L.DistSolver(lat, cfg.eps, a, b, c, p, cfg.sigma, world=world, rank=rank, device=local,
                         nccl_id=uid[0], norm2=norm2)
        G = world
    else:
        G = max(1, args.virtual_ranks)
        D = L.DistSolver(lat, cfg.eps, a, b, c, p, cfg.sigma, world=G, rank=-1, device=0, norm2=norm2)
    D.set_dt(cfg.dt)
    D.discretize_initial()
    m = cfg.m if args.m is None else args.m
    for _ in range(args.warmup):
        D.step(m)
    barrier(dist)
    per = [D.time_steps(m) for _ in range(args.steps)]
    barrier(dist)
    total_ms = max_over_ranks(sum(per), dist, torch)
    norm = D.l2_norm()
    info = D.info()
    # per-rank algorithmic bytes per Strang step: COL pass R+W
    # of the column slab + V; row side R+W of the row slab per local pass
    # (1, or 3 for three-level rows) + K^; exchanges: 2 per step, each rank
    # sending (G-1) blocks of M/G^2 elements over NVLink
    slab = info["M"] / G
    row_passes = 3 if info.get("Ma", 0) else 1
    hbm = 32.0 * slab + 16.0 * slab + row_passes * 32.0 * slab + 16.0 * slab
    nvl = 2.0 * 16.0 * info["M"] * (G - 1) / (G * G)
    t_roof = hbm / (measured_hbm_peak()[0] * 1e9) + (nvl / 900e9 if world > 1 else 0.0)
    t_meas = 1e-3 * total_ms / (args.steps * m)
    if rank == 0:
        line = {
            "metric": METRIC, "value": float(cfg.N) * m * args.steps / (total_ms * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (complex fp64)",
            "data": "synthetic (seeded BASELINE families, DESIGN.md Seeds)",
            "config": {**config_dict(cfg, args), "parallelism": f"one wave function sharded over {G} ranks "
                       f"({'NCCL send/recv' if world > 1 else 'virtual ranks on one GPU, device copies'}), "
                       "2 block exchanges per Strang step"},
            "sharded": {**info, "ranks": G, "norm_after": norm},
            "roofline": {"bound": "hbm+nvlink", "hbm_bytes_per_rank_step": hbm, "nvlink_bytes_per_rank_step": nvl,
                         "t_roof_us": 1e6 * t_roof, "frac": t_roof / t_meas,
                         "note": "virtual ranks share one GPU's HBM: the exchange is device copies, not NVLink"
                         if world == 1 else "HBM at MEASURED_PEAKS hbm_gbs, NVLink 900 GB/s per direction"},
            "us_per_strang_step": 1e3 * total_ms / (args.steps * m),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1")
    ap.add_argument("--method", default="circulant", choices=["circulant", "bluestein"])
    ap.add_argument("--batch", type=int, default=None, help="ensemble members (C3); default: the config's")
    ap.add_argument("--m", type=int, default=None, help="Strang steps per bench step (default: the config's m)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-sample-steps", type=int, default=4)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", action="store_true", help="shard one wave function across the ranks (NCCL)")
    ap.add_argument("--virtual-ranks", type=int, default=0, help="sharded path with G virtual ranks on one GPU")
    args = ap.parse_args()
    from paper_1808_06357_b200 import configs

    cfg = configs.CONFIGS[args.config]
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the timing rules ask for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.shard or args.virtual_ranks > 0:
        return run_sharded(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
