"""Radix-plan search for the pass kernels: for each line length, every
ordered factorisation into compiled radices with the current number of
stages and no larger maximum radix, scored by the shared-memory wavefront
model (smem_sim.py, quarter-warp bank groups, calibrated against ncu). Prints
the kPlanOverride rows of fft_core.cuh.

    python plan_search.py 486 1080 ...
"""
import itertools
import sys

import smem_sim as S

RADICES = [2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 15, 16, 18, 20, 21, 24, 27, 28, 32]
_orig = S.wavefronts


def _quarter(addrs):
    return sum(_orig(addrs[k:k + 8]) for k in range(0, len(addrs), 8))


S.wavefronts = _quarter


def factorizations(L, n):
    if n == 1:
        return [[L]] if L in RADICES else []
    out = []
    for r in RADICES:
        if L % r == 0 and L // r > 1:
            for rest in factorizations(L // r, n - 1):
                out.append([r] + rest)
    return out


def geometry(L, axis):
    if axis == "ROW":
        B = 1 if L >= 256 else 256 // L
    else:
        B = 1 if L >= 8192 else (2 if (L >= 512 and L != 512) else (4 if L >= 128 else 8))
    return B


def nt_for(L, B, plan, axis):
    raw = B * max(L // r for r in plan)
    if axis == "COL" and L >= 4096 or (axis == "COL" and L == 512):
        return 256
    return 32 if raw <= 32 else (512 if raw >= 512 else ((raw + 31) // 32) * 32)


def score(L, axis, plan):
    B = geometry(L, axis)
    NT = nt_for(L, B, plan, axis)
    swz = (plan[0] % 2 == 0 or plan[-1] % 2 == 0) and L >= 16
    wf, _ = S.simulate(L, axis, B, NT, plan, swz)
    util = sum(B * (L // r) for r in plan) / (len(plan) * NT * -(-max(B * (L // r) for r in plan) // NT))
    return wf / (B * L), NT, swz, util


def best(L, axis, cur):
    cands = [p for p in factorizations(L, len(cur)) if max(p) <= max(cur)]
    rows = []
    for p in cands:
        w, NT, swz, util = score(L, axis, p)
        rows.append((round(w, 3), -round(util, 2), p, NT, swz))
    rows.sort()
    return rows


if __name__ == "__main__":
    for tok in sys.argv[1:]:
        L, axis, cur = tok.split(":")
        L = int(L)
        cur = [int(x) for x in cur.split(",")]
        w, NT, swz, util = score(L, axis, cur)
        print(f"L={L} {axis} current {cur} NT={NT} swz={swz}: {w:.3f} wf/elem, util {util:.2f}")
        for r in best(L, axis, cur)[:5]:
            print("    ", r)
