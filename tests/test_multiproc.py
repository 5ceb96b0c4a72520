"""Multi-process host logic on CPU (gloo, world_size 2).

Config 3 shards its 512 independent members across ranks with no data-path
collective; each rank steps configs.shard_members(...) and
only the final observables are gathered. Here every rank runs the CPU oracle
on its shard of a small ensemble and the all-gathered result must equal the
single-process run member for member; bench.py's max-over-ranks timing
reduction is exercised the same way.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ensemble(batch):
    import sys

    sys.path.insert(0, ROOT)
    import paper_1808_06357_b200 as L
    from paper_1808_06357_b200 import configs

    lat, a, b, c, p = configs.small_rank1(3, 257, seed=31, batch=batch, c_range=(0.3, 0.7), p_max=3)
    norm2, _, _ = L.aaset_build(lat, with_vectors=False)
    return lat, norm2, a, b, c, p


def _run_members(lat, norm2, a, b, c, p, members, steps=5):
    from oracle.pyoracle import Oracle

    gen, moduli = lat.generators()
    orc = Oracle(gen, moduli, norm2, 0.05, a, b)
    orc.set_dt(1.0 / 64)
    out = []
    for m in members:
        u = orc.analyze(orc.initial_samples(c[m], p[m], 0.1))
        out.append(orc.steps(u, steps))
    return np.array(out)


def _worker(rank, world, port, batch, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1808_06357_b200 import configs

    import bench

    lat, norm2, a, b, c, p = _ensemble(batch)
    m0, cnt = configs.shard_members(batch, rank, world)
    mine = _run_members(lat, norm2, a, b, c, p, range(m0, m0 + cnt))
    # gather variable-size shards (pad to the largest)
    n = lat.n_total()
    pad = np.zeros((batch // world + 1, n), np.complex128)
    pad[:cnt] = mine
    t = torch.from_numpy(pad.view(np.float64).copy())
    bufs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)
    # bench's timing reduction: max over ranks
    tmax = bench.reduce_over_ranks(float(rank + 1) * 1.5, dist, torch)
    if rank == 0:
        full = []
        for r in range(world):
            _, cr = configs.shard_members(batch, r, world)
            full.append(bufs[r].numpy().view(np.complex128)[:cr])
        q.put((np.concatenate(full), tmax))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [4, 5])
def test_gloo_two_rank_ensemble_matches_single_process(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got, tmax = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    lat, norm2, a, b, c, p = _ensemble(batch)
    want = _run_members(lat, norm2, a, b, c, p, range(batch))
    assert got.shape == want.shape
    assert np.array_equal(got, want)  # same arithmetic per member: bit-identical
    assert tmax == 3.0


def test_bench_reference_arm_under_torchrun_two_ranks():
    """bench.py --impl reference launched like the driver's N>1 arm
    (torch.distributed.run, two ranks, gloo here): rank 0 alone runs and
    prints ONE JSON line, the other rank exits 0 without work."""
    import json
    import subprocess
    import sys

    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference",
           "--gpus", "2", "--config", "C0", "--steps", "2", "--warmup", "1", "--ref-seconds", "0.2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 2
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_respawns_ranks_without_launcher(monkeypatch):
    """`bench.py --gpus N` with no WORLD_SIZE re-launches itself through
    torch.distributed.run with N processes on 127.0.0.1."""
    import sys

    import bench

    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    bench.main()
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
