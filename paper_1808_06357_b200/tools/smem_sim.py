"""Shared-memory wavefront model of one fused pass (fft_pass.cuh): replays
every stage's smem reads and writes per warp instruction and counts
wavefronts (max distinct 16-byte addresses per 4-bank group, >= 1 per 8
active lanes). Used to pick radix plans / layouts without a GPU; calibrated
against ncu's l1tex__data_pipe_lsu_wavefronts_mem_shared (profiles/r2).

    python smem_sim.py 486 ROW 1 96 9,9,6 [swz]
"""
import sys
from collections import Counter


def wavefronts(addrs):
    """addrs: 16-byte slot indices of the active lanes of one warp instruction."""
    if not addrs:
        return 0
    groups = {}
    for a in set(addrs):
        groups.setdefault(a % 8, set()).add(a)
    return max(max(len(v) for v in groups.values()), (len(addrs) + 7) // 8)


def simulate(L, axis, B, NT, plan, swizzle, pad=None):
    phys = (lambda i: i + (i >> 4)) if swizzle else (lambda i: i)
    span = phys(L - 1) + 1
    if pad is None:
        if B == 1:
            pad = 0
        else:
            want = 2 if B == 4 else (4 if B == 2 else 1)
            pad = ((want - span % 8) % 8 + 8) % 8
    LS = span + pad
    slot = lambda b, i: b * LS + phys(i)
    nst = len(plan)

    def stage_ns(pl, s):
        p = 1
        for x in pl[:s]:
            p *= x
        return p

    def mapq(q, T):
        return (q // T, q % T) if axis == "ROW" else (q % B, q // B)

    total = 0
    detail = []
    # sequence of (kind, plan, stage): T1 stages 0..nst-2 (write), mid (read T1 last, write T2 first), T2 stages 1..nst-1
    rev = plan[::-1]
    ops = []
    for s in range(nst):
        R = plan[s]; T = L // R; Ns = stage_ns(plan, s)
        if s > 0:
            ops.append(("read", R, T, None))
        if s < nst - 1:
            ops.append(("write", R, T, Ns))
    # mid: T1 last stage read (above), T2 first stage write j*R + r
    ops.append(("write_mid", rev[0], L // rev[0], 1))
    for s in range(1, nst):
        R = rev[s]; T = L // R; Ns = stage_ns(rev, s)
        ops.append(("read", R, T, None))
        if s < nst - 1:
            ops.append(("write", R, T, Ns))
    for kind, R, T, Ns in ops:
        tasks = B * T
        tpt = (tasks + NT - 1) // NT
        wf = 0
        for t in range(tpt):
            for w in range(0, NT, 32):
                for r in range(R):
                    addrs = []
                    for lane in range(32):
                        q = w + lane + t * NT
                        if q >= tasks:
                            continue
                        b, j = mapq(q, T)
                        if kind == "read":
                            i = j + r * T
                        elif kind == "write_mid":
                            i = j * R + r
                        else:
                            i = (j // Ns) * Ns * R + j % Ns + r * Ns
                        addrs.append(slot(b, i))
                    wf += wavefronts(addrs)
        detail.append((kind, R, Ns, wf))
        total += wf
    return total, detail


if __name__ == "__main__":
    L = int(sys.argv[1]); axis = sys.argv[2]; B = int(sys.argv[3]); NT = int(sys.argv[4])
    plan = [int(x) for x in sys.argv[5].split(",")]
    swz = len(sys.argv) > 6 and sys.argv[6] == "swz"
    tot, det = simulate(L, axis, B, NT, plan, swz)
    ideal = 2 * (len(plan) - 1) * 2 * B * L // 8 // 2 * 2
    print(f"L={L} {axis} B={B} NT={NT} plan={plan} swz={swz}: {tot} wavefronts per tile "
          f"({tot / (B * L):.3f} per element; ideal {(2 * len(plan)) * B * L / 8 / (B * L):.3f})")
    for d in det:
        print("   ", d)
