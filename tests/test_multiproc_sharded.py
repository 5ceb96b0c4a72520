"""Sharded four-step convolution across processes (CPU, gloo): the exact data
distribution of paper_1808_06357_b200/csrc/cuda/solver_dist.cu -- column
slabs of width Wb = M2/G, block-major row slabs of height Hb = M1/G,
contiguous (Hb x Wb) block exchanges by grouped point-to-point send/recv
(the NCCL path's pattern) -- restated in numpy and checked against a
single-process length-M cyclic convolution. The device kernels of the same
path are covered on one GPU with virtual ranks (tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(M1, M2, seed=0):
    rng = np.random.default_rng(seed)
    M = M1 * M2
    z = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    Khat = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    return z, Khat


def _exchange(send_blocks, world, rank):
    """send_blocks[h] goes to rank h; returns recv[h] from rank h."""
    recv = [np.empty_like(send_blocks[rank]) for _ in range(world)]
    reqs = []
    for h in range(world):
        if h == rank:
            recv[h] = send_blocks[h].copy()
            continue
        sb = torch.from_numpy(send_blocks[h].view(np.float64).copy())
        rb = torch.empty_like(sb)
        reqs.append((dist.isend(sb, h), dist.irecv(rb, h), h, rb))
    for s, r, h, rb in reqs:
        s.wait()
        r.wait()
        recv[h] = rb.numpy().view(np.complex128).reshape(send_blocks[rank].shape)
    return recv


def _worker(rank, world, port, M1, M2, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z, Khat = _problem(M1, M2)
    M = M1 * M2
    Hb, Wb = M1 // world, M2 // world
    Z = z.reshape(M1, M2)
    cols = np.arange(rank * Wb, (rank + 1) * Wb)
    # column slab: forward column FFT + four-step twiddle with GLOBAL column index
    A = np.fft.fft(Z[:, cols], axis=0) * np.exp(-2j * np.pi * np.outer(np.arange(M1), cols) / M)
    # col -> row exchange: block h = rows of rank h (contiguous in the slab)
    recv = _exchange([A[h * Hb:(h + 1) * Hb, :] for h in range(world)], world, rank)
    B = np.concatenate(recv, axis=1)  # rows [rank*Hb, ...), all M2 columns
    rows = np.arange(rank * Hb, (rank + 1) * Hb)
    Kb = Khat.reshape(M2, M1).T[rows, :]  # ROW-pass order: X[k1 + M1 k2] at (k1, k2)
    B = np.fft.ifft(np.fft.fft(B, axis=1) * Kb, axis=1) * M2
    # row -> col exchange: block g = columns of rank g
    back = _exchange([B[:, g * Wb:(g + 1) * Wb] for g in range(world)], world, rank)
    A = np.concatenate(back, axis=0)  # all M1 rows, my columns
    A = np.fft.ifft(A * np.exp(2j * np.pi * np.outer(np.arange(M1), cols) / M), axis=0) * M1
    q.put((rank, A))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M1,M2,world", [(6, 8, 2), (12, 9, 3)])
def test_sharded_fourstep_convolution(M1, M2, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M1, M2, q)) for r in range(world)]
    for p in procs:
        p.start()
    slabs = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    z, Khat = _problem(M1, M2)
    want = np.fft.ifft(np.fft.fft(z) * Khat) * (M1 * M2)  # unnormalised IFFT(FFT(z) K^)
    Wb = M2 // world
    got = np.zeros((M1, M2), complex)
    for r, A in slabs.items():
        got[:, r * Wb:(r + 1) * Wb] = A
    assert np.abs(got.reshape(-1) - want).max() <= 1e-10 * np.abs(want).max()


def _worker3(rank, world, port, M1, Ma, Mb, q):
    """Three-level rows (config 4's layout): each length-M2 row is an Ma x Mb
    matrix. The row slab is kept in the device's block-major MEMORY order and
    addressed exactly as the kernels do (PassArgs rb_w / rb_stride, batch =
    slab row), so this restates solver_dist.cu's three local row passes."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    M2 = Ma * Mb
    z, Khat = _problem(M1, M2)
    M = M1 * M2
    Hb, Wb = M1 // world, M2 // world
    Z = z.reshape(M1, M2)
    cols = np.arange(rank * Wb, (rank + 1) * Wb)
    A = np.fft.fft(Z[:, cols], axis=0) * np.exp(-2j * np.pi * np.outer(np.arange(M1), cols) / M)
    recv = _exchange([A[h * Hb:(h + 1) * Hb, :] for h in range(world)], world, rank)
    mem = np.stack(recv).reshape(-1)  # block q (from rank q) = Hb x Wb, block-major
    # COL pass of length Ma inside slab row r (fft_pass.cuh Ctx::pos, AX_COL with rb_w):
    # p = ia*Mb + ib, q = p / Wb, address = r*Wb (batch) + q*Hb*Wb + p % Wb
    r_, ia, ib = np.meshgrid(np.arange(Hb), np.arange(Ma), np.arange(Mb), indexing="ij")
    p = ia * Mb + ib
    addr = r_ * Wb + (p // Wb) * (Hb * Wb) + p % Wb
    assert np.array_equal(mem[addr], np.concatenate(recv, axis=1).reshape(Hb, Ma, Mb))
    tw = np.exp(-2j * np.pi * np.outer(np.arange(Ma), np.arange(Mb)) / M2)  # W_M2^(ka*ib)
    mem[addr] = np.fft.fft(mem[addr], axis=1) * tw
    # ROW pass of length Mb: the slab is Hb*Ma contiguous Mb-lines (Mb | Wb)
    pos = np.zeros((M1, M2), complex)  # K^ in ROW-pass order: (k1, ka*Mb + kb) holds X[k1 + M1 (ka + Ma kb)]
    k1, ka, kb = np.meshgrid(np.arange(M1), np.arange(Ma), np.arange(Mb), indexing="ij")
    pos[k1, ka * Mb + kb] = Khat[k1 + M1 * (ka + Ma * kb)]
    rows = np.arange(rank * Hb, (rank + 1) * Hb)
    Kslab = np.stack([pos[rows, g * Wb:(g + 1) * Wb] for g in range(world)]).reshape(-1, Mb)  # k_rowblk
    lines = mem.reshape(-1, Mb)
    mem = (np.fft.ifft(np.fft.fft(lines, axis=1) * Kslab, axis=1) * Mb).reshape(-1)
    mem[addr] = np.fft.ifft(mem[addr] * np.conj(tw), axis=1) * Ma
    blocks = mem.reshape(world, Hb, Wb)
    back = _exchange([blocks[g] for g in range(world)], world, rank)
    A = np.concatenate(back, axis=0)
    A = np.fft.ifft(A * np.exp(2j * np.pi * np.outer(np.arange(M1), cols) / M), axis=0) * M1
    q.put((rank, A))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M1,Ma,Mb,world", [(4, 6, 5, 2), (6, 6, 4, 3)])
def test_sharded_three_level_convolution(M1, Ma, Mb, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker3, args=(r, world, port, M1, Ma, Mb, q)) for r in range(world)]
    for p in procs:
        p.start()
    slabs = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    M2 = Ma * Mb
    z, Khat = _problem(M1, M2)
    want = np.fft.ifft(np.fft.fft(z) * Khat) * (M1 * M2)
    Wb = M2 // world
    got = np.zeros((M1, M2), complex)
    for r, A in slabs.items():
        got[:, r * Wb:(r + 1) * Wb] = A
    assert np.abs(got.reshape(-1) - want).max() <= 1e-10 * np.abs(want).max()
