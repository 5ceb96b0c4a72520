"""Benchmark of the Strang time-stepping hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C3] [--method circulant|bluestein]

Workload (config.workload): BASELINE.json configs[3] = C3, the configuration
the metric ("... 1/2/4/8 B200") is quoted on and the largest that runs on one
GPU: 512 independent wave functions, d=6 rank-1 lattice, N = 262147 (smallest
prime >= 2^18), eps=0.05, T=0.5, m=512, shared z and v. One bench step = one
full propagation (m = 512 Strang steps) of every member.
L2 is flushed (512 MiB memset) before every timed bench step, outside its
event pair; a member group's working set (4.3 GB) is far beyond L2 anyway.

value    : lattice-point Strang steps/s = N * members * m * K / (max over ranks
           of the summed device time of the K steps), CUDA events on the solver
           stream. --gpus N shards the 512 members over N ranks (no data-path
           collective); without WORLD_SIZE in the environment
           bench.py launches the N ranks itself through torch.distributed.run.
e2e      : the same metric through the public API with host buffers: per step
           set_state from pinned host memory (H2D), step(m), get_state (D2H),
           wall clock around the synchronous calls, max over ranks.
roofline : dominant pass kernel, algorithmic bytes per launch (every member's
           state read and written once + the shared diagonal table once) / its
           average event-timed duration, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: rank 0 at N=1 only, bounded samples on this host's cores: the
           oracle's literal Strang step with scipy.fft (pocketfft) transforms
           on all threads (the value), plus single-thread, circulant-form and
           C++-oracle datapoints (oracle/, a port of the reference's specified
           solver -- the reference itself has no solver).
--impl reference: that CPU port on all host threads, rank 0 only, inputs from
           oracle/ alone (oracle/cases.py lattices and seeds, the oracle's own
           shell-walk norm table) -- nothing from the product package.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
        else:
            dist.init_process_group("gloo")
        return world, rank, local, dist, torch
    return 1, 0, 0, None, None


def _dev(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def reduce_over_ranks(x, dist, torch, op="max"):
    if dist is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def respawn(n):
    """`bench.py --gpus N` without a launcher: run N ranks through
    torch.distributed.run (one process per GPU), rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ CPU port
CPU_MAX_N = 1 << 25  # the CPU port runs configs up to this size; C4 uses C4r


def cpu_case(name):
    """(case, norm table, note) from oracle/ only: the config's lattice and
    seeds restated in oracle/cases.py, the oracle's own shell-walk norm table.
    Config 4 (17 GB per state) uses its reduced-N twin C4r."""
    from oracle import pyoracle as po
    from oracle.cases import CASES

    note = ""
    if name == "C4":
        name = "C4r"
        note = " (C4r: config 4's shape at N = 16777259; the full-N CPU step does not fit a bounded sample)"
    cs = CASES[name]
    if not cs.gen[0]:
        raise RuntimeError(f"{name}: no oracle-side generating vector")
    norm2, _ = po.aaset(cs.gen, cs.moduli, with_vectors=False)
    return cs, norm2, note


class CpuPort:
    """Bounded CPU samples of the workload (oracle/ only)."""

    def __init__(self, name, workers=None):
        from oracle import pyoracle as po
        from oracle.scipy_port import ScipyPort

        self.cs, norm2, self.note = cpu_case(name)
        a, b, _ = self.cs.potential_params()
        self.orc = po.Oracle(self.cs.gen, self.cs.moduli, norm2, self.cs.eps, a, b)
        self.orc.set_dt(self.cs.dt)
        self.port = ScipyPort(self.orc, self.cs.moduli, norm2, self.cs.eps, workers=workers)
        self.port.set_dt(self.cs.dt)
        c, p = self.cs.member(0)
        self.g = self.orc.initial_samples(c, p, self.cs.sigma)
        self.u = self.orc.analyze(self.g)

    def rate(self, kind, steps):
        """lattice-pt-steps/s of `steps` Strang steps of one wave function."""
        t0 = time.perf_counter()
        if kind == "literal":
            self.port.steps(self.u, steps)
        elif kind == "circulant":
            self.port.circulant_steps(self.port.potH * self.g, steps)
        elif kind == "oracle":
            self.orc.steps(self.u, steps)
        dt = time.perf_counter() - t0
        return self.cs.N * steps / dt, dt

    def sized(self, kind, seconds):
        r1, t1 = self.rate(kind, 1)
        steps = max(1, min(self.cs.m, int(seconds / max(t1, 1e-4))))
        return steps


def oracle_single_thread_rate(name, seconds):
    """The C++ oracle on ONE thread, in a child process (OMP_NUM_THREADS=1)."""
    code = ("import sys,json; sys.path.insert(0, %r); import bench; p = bench.CpuPort(%r, workers=1); "
            "n = p.sized('oracle', %f); r, t = p.rate('oracle', n); print(json.dumps([r, n, t]))") % (ROOT, name, seconds)
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=900)
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline(name, seconds):
    cores = os.cpu_count()
    p = CpuPort(name)
    n = p.sized("literal", seconds)
    rate, t = p.rate("literal", n)
    p1 = CpuPort(name, workers=1)
    n1 = p1.sized("literal", seconds / 2)
    rate1, t1 = p1.rate("literal", n1)
    extra = {"literal_1_thread": {"value": rate1, "steps": n1, "seconds": t1}}
    if len(p.cs.moduli) == 1:
        nc = p.sized("circulant", seconds / 2)
        rc, tc = p.rate("circulant", nc)
        extra["circulant_all_threads"] = {"value": rc, "steps": nc, "seconds": tc,
                                          "note": "same operator as one length-M cyclic convolution per step"}
    no = p.sized("oracle", seconds / 2)
    ro, to = p.rate("oracle", no)
    extra["cxx_oracle_all_threads"] = {"value": ro, "steps": no, "seconds": to,
                                       "note": "oracle.cpp's own recursive FFT + Bluestein, OpenMP"}
    try:
        r, nn, tt = oracle_single_thread_rate(name, seconds / 2)
        extra["cxx_oracle_1_thread"] = {"value": r, "steps": nn, "seconds": tt}
    except Exception as e:  # noqa: BLE001
        extra["cxx_oracle_1_thread"] = {"error": str(e)[:200]}
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"{n} literal Strang steps (SPEC.md:336-344) of one {p.cs.name} wave function, oracle setup + "
                      f"scipy.fft transforms on {cores} threads, {t:.1f} s{p.note}",
            "datapoints": extra}


def run_reference(args):
    world, rank, _, dist, torch = dist_setup()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    cores = os.cpu_count()
    p = CpuPort(args.config)
    sample = p.sized("literal", args.ref_seconds)
    for _ in range(args.warmup):
        p.rate("literal", 1)
    rates, times = [], []
    for _ in range(args.steps):
        r, t = p.rate("literal", sample)
        rates.append(r)
        times.append(t)
    value = p.cs.N * sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128 (complex fp64)",
        "data": "synthetic (seeded BASELINE families, oracle/cases.py)",
        "config": config_dict(args, note=f"1 reference step = {sample} Strang steps of one wave function "
                                          "(bounded sample); rate per lattice-point step"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"{sample} literal Strang steps of one {p.cs.name} wave function per bench step "
                                   f"(4 length-N DFTs each, scipy.fft on {cores} threads){p.note}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def config_dict(args, note=None, world=1):
    from oracle.cases import CASES  # plain data; the same table as configs.py (tests/test_oracle_cases.py)

    cs = CASES.get(args.config)
    if cs is None:
        wl = args.config
    else:
        wl = (f"{cs.name}: d={cs.d} rank-{len(cs.moduli)} N={cs.N} eps={cs.eps} T={cs.T} m={cs.m} "
              f"members={cs.batch}; 1 bench step = full propagation (m Strang steps) of every member")
    d = {"workload": wl, "method": args.method,
         "l2": "flushed (512 MiB memset) before every timed bench step; per-pass working set >> L2",
         "parallelism": ("1 GPU" if world == 1 else f"{world} GPUs: ensemble members sharded by rank "
                         "(configs.shard_members), no data-path collective")}
    if note:
        d["note"] = note
    return d


# ------------------------------------------------------------------ our arm
def traffic_for(cfg_name, method, side, info):
    """ncu DRAM bytes per launch from profiles/ncu_traffic.json, only when the
    entry was captured on this geometry and kernel family (else null)."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        e = json.load(open(tp)).get(f"{cfg_name}_{method}_{side}")
    except Exception:
        return None, None
    if not isinstance(e, dict):
        return None, None
    want = {"M1": info["M1"], "M2": info["M2"], "group": info["group"], "kernel": info.get("pass_kernel")}
    if any(e.get(k) != v for k, v in want.items()):
        return None, None
    return e["bytes"], e.get("source")


def run_ours(args):
    world, rank, local, dist, torch = dist_setup()
    import paper_1808_06357_b200 as L
    from paper_1808_06357_b200 import configs

    cfg = configs.CONFIGS[args.config]
    lat = configs.lattice(cfg)
    batch_total = cfg.batch if args.batch is None else args.batch
    a, b, c, p = configs.problem(cfg, batch=batch_total)
    if batch_total > 1:
        m0, batch = configs.shard_members(batch_total, rank, world)
        c, p = c[m0:m0 + batch], p[m0:m0 + batch]
        members_all = batch_total
    else:
        batch = 1  # a single wave function: every rank runs a replica
        members_all = world
    norm2 = None if cfg.rank == 1 else L.aaset_build(lat, with_vectors=False)[0]
    S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma, method=args.method, device=local, norm2=norm2)
    S.set_dt(cfg.dt)
    S.discretize_initial()
    m = cfg.m if args.m is None else args.m

    for _ in range(args.warmup):
        S.step(m)
    info = S.info()  # after the warm-up: pass_kernel reports what the steps ran on

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
    total_ms = reduce_over_ranks(sum(per_step), dist, torch)
    work = float(cfg.N) * members_all * m * args.steps
    value = work / (total_ms * 1e-3)

    # ---- per-pass durations (event-timed launches on the solver stream)
    S.flush_l2()
    ms_col, ms_row = S.profile_passes(min(m, 64))
    peak, peak_kind = measured_hbm_peak()
    groups = -(-batch // max(1, info["group"]))
    pass_bytes = {"col": info["bytes_per_pass_col"] / groups, "row": info["bytes_per_pass_row"] / groups}
    pass_ms = {"col": ms_col, "row": ms_row}
    dom = "col" if ms_col >= ms_row else "row"
    achieved = pass_bytes[dom] / (pass_ms[dom] * 1e-3) / 1e9
    traffic, tsrc = traffic_for(cfg.name, args.method, dom, info)
    step_ms = statistics.mean(per_step) / m
    step_bytes = info["bytes_per_step"]  # all members of this rank, every pass of one Strang step
    canonical = ((160.0 * info["M"] + 18.0 * info["n_total"]) * batch if cfg.rank == 1
                 else 82.0 * info["n_total"] * batch)
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "traffic_source": tsrc,
        "kernel": f"{dom} pass ({info.get('pass_kernel', 'fft_pass')}, {'COL' if dom == 'col' else 'ROW'} axis)",
        "bytes_per_launch": pass_bytes[dom], "avg_launch_ms": pass_ms[dom], "peak_kind": peak_kind,
        "bytes_model": "every member's state read+written once per pass (32 B x M per member) + the shared "
                       "diagonal table once per launch (V: 16 N, K^: 16 M)",
        "passes": {s: {"ms": pass_ms[s], "bytes": pass_bytes[s],
                       "frac": pass_bytes[s] / (pass_ms[s] * 1e-3) / 1e9 / peak} for s in ("col", "row")},
        "step": {"bytes": step_bytes, "us": step_ms * 1e3,
                 "frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak},
        "extra_canonical_model": {
            "note": "NOT a roofline fraction: SURVEY.md 8(d)'s literal 4-pass Bluestein bytes (160 M + 18 N per "
                    "member) over the measured time of our 2-pass circulant step (an algorithm credit)",
            "canonical_bytes_per_step": canonical, "t_roof_us_at_8TBps": canonical / 8e12 * 1e6},
    }

    # ---- e2e through the public API with pinned host buffers
    import torch as _t

    n = cfg.N * batch
    host_in = _t.empty(2 * n, dtype=_t.float64, pin_memory=_t.cuda.is_available())
    host_out = _t.empty(2 * n, dtype=_t.float64, pin_memory=_t.cuda.is_available())
    g = S.get_state()
    host_in.numpy()[:] = g.reshape(-1).view(np.float64)
    e2e_times = []
    barrier(dist)
    for _ in range(args.steps):
        S.flush_l2()
        t0 = time.perf_counter()
        S.set_state_ptr(host_in.data_ptr(), batch)
        S.step(m)
        S.get_state_ptr(host_out.data_ptr(), batch)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = reduce_over_ranks(sum(e2e_times), dist, torch)
    e2e = {"value": float(cfg.N) * members_all * m * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": 16 * cfg.N * members_all, "d2h_bytes_per_step": 16 * cfg.N * members_all,
           "ms_per_step": 1e3 * e2e_s / args.steps}

    # ---- CPU baseline (rank 0, N=1 only): oracle ports, bounded samples
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(cfg.name, args.cpu_seconds)
        except Exception as e:  # noqa: BLE001
            cpu = {"error": str(e)[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if batch_total > 1 else "weak", "vs_baseline": None, "dtype": "c128 (complex fp64)",
            "data": "synthetic (seeded BASELINE families, DESIGN.md Seeds)",
            "config": config_dict(args, world=world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(reduce_over_ranks(launches, dist, torch, "sum")), "clocks": clk,
            "solver": {k: info[k] for k in ("M", "M1", "M2", "group", "launches_per_step", "bytes_per_step")
                       if k in info} | {"members_per_rank": batch, "pass_kernel": info.get("pass_kernel")},
            "us_per_strang_step": step_ms * 1e3,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- sharded arm
def run_sharded(args):
    """One wave function sharded over the ranks (DistSolver): NCCL exchanges
    between GPUs under torchrun, or --virtual-ranks G on one GPU."""
    world, rank, local, dist, torch = dist_setup()
    import paper_1808_06357_b200 as L
    from paper_1808_06357_b200 import configs

    cfg = configs.CONFIGS[args.config]
    lat = configs.lattice(cfg)
    a, b, c, p = configs.problem(cfg, batch=1)
    if world > 1:
        uid = [L.DistSolver.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        D = L.DistSolver(lat, cfg.eps, a, b, c, p, cfg.sigma, world=world, rank=rank, device=local, nccl_id=uid[0])
        G = world
    else:
        G = max(1, args.virtual_ranks)
        D = L.DistSolver(lat, cfg.eps, a, b, c, p, cfg.sigma, world=G, rank=-1, device=0)
    D.set_dt(cfg.dt)
    D.discretize_initial()
    m = cfg.m if args.m is None else args.m
    for _ in range(args.warmup):
        D.step(m)
    barrier(dist)
    per = [D.time_steps(m) for _ in range(args.steps)]
    barrier(dist)
    total_ms = reduce_over_ranks(sum(per), dist, torch)
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
    t_roof = hbm / (measured_hbm_peak()[0] * 1e9) + (nvl / 770e9 if world > 1 else 0.0)
    t_meas = 1e-3 * total_ms / (args.steps * m)
    if rank == 0:
        line = {
            "metric": METRIC, "value": float(cfg.N) * m * args.steps / (total_ms * 1e-3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (complex fp64)",
            "data": "synthetic (seeded BASELINE families, DESIGN.md Seeds)",
            "config": {**config_dict(args, world=world), "parallelism": f"one wave function sharded over {G} ranks "
                       f"({'NCCL send/recv' if world > 1 else 'virtual ranks on one GPU, device copies'}), "
                       "2 block exchanges per Strang step"},
            "sharded": {**info, "ranks": G, "norm_after": norm},
            "roofline": {"bound": "hbm+nvlink", "hbm_bytes_per_rank_step": hbm, "nvlink_bytes_per_rank_step": nvl,
                         "t_roof_us": 1e6 * t_roof, "frac": t_roof / t_meas,
                         "note": "virtual ranks share one GPU's HBM: the exchange is device copies, not NVLink"
                         if world == 1 else "HBM at MEASURED_PEAKS hbm_gbs, NVLink at the measured 770 GB/s"},
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
    ap.add_argument("--config", default="C3")
    ap.add_argument("--method", default="circulant", choices=["circulant", "bluestein"])
    ap.add_argument("--batch", type=int, default=None, help="ensemble members (C3); default: the config's")
    ap.add_argument("--m", type=int, default=None, help="Strang steps per bench step (default: the config's m)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0, help="CPU baseline: seconds per datapoint")
    ap.add_argument("--ref-seconds", type=float, default=3.0, help="reference arm: seconds per bench step")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", action="store_true", help="shard one wave function across the ranks (NCCL)")
    ap.add_argument("--virtual-ranks", type=int, default=0, help="sharded path with G virtual ranks on one GPU")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return respawn(args.gpus)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the timing rules ask for >= 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    if args.shard or args.virtual_ranks > 0:
        return run_sharded(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
