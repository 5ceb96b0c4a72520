"""Shared-memory wavefronts of the pass4 stage sequence (fft_pass4.cuh) for a
line length and radix plan: 16-byte accesses are served per quarter warp
(8 lanes), one wavefront per distinct 128-byte bank row set -- a quarter warp
costs max over the eight 16-byte bank groups of the distinct addresses in it.
Usage: python p4_conflicts.py L r0 r1 r2 [axis B LS]"""
import sys
from collections import defaultdict


def qw_cost(addrs):
    groups = defaultdict(set)
    for a in addrs:
        groups[a % 8].add(a)
    return max(len(s) for s in groups.values())


def stage_cost(tasks_addr, nt, R):
    """tasks_addr(q, r) -> slot or None; returns (wavefronts, ideal)"""
    tot = ideal = 0
    for r in range(R):
        for w0 in range(0, nt, 8):
            ad = [tasks_addr(q, r) for q in range(w0, w0 + 8)]
            ad = [a for a in ad if a is not None]
            if ad:
                tot += qw_cost(ad)
                ideal += 1
    return tot, ideal


def analyze(L, plan, axis="row", B=1, LS=None, verbose=True):
    LS = LS or L
    nst = len(plan)
    seq = []  # (R, Ns, kind) over the pass: fwd stages, mid, reversed stages
    ns = 1
    for s, R in enumerate(plan):
        seq.append((R, ns, "first" if s == 0 else ("mid" if s == nst - 1 else "inner")))
        ns *= R
    rev = plan[::-1]
    ns = rev[0]
    for s in range(1, nst):
        seq.append((rev[s], ns, "last" if s == nst - 1 else "inner"))
        ns *= rev[s]
    total = ideal = 0
    for (R, Ns, kind) in seq:
        T = L // R
        ntask = B * T

        def dec(q):
            if q >= ntask:
                return None
            return (q // T, q % T) if axis == "row" else (q % B, q // B)

        def rd(q, r):
            d = dec(q)
            return None if d is None else d[0] * LS + d[1] + r * T

        def wr(q, r, Ns=Ns, R=R):
            d = dec(q)
            if d is None:
                return None
            b, j = d
            k = j % Ns
            return b * LS + (j - k) * R + k + r * Ns

        def wr0(q, r, R=R):  # Ns = 1 writes (first stage, mid stage's second transform)
            d = dec(q)
            return None if d is None else d[0] * LS + d[1] * R + r

        nt = ((ntask + 31) // 32) * 32
        parts = []
        if kind != "first":
            parts.append(("rd", stage_cost(rd, nt, R)))
        if kind == "first" or kind == "mid":
            parts.append(("wr", stage_cost(wr0, nt, R)))
        elif kind == "inner":
            parts.append(("wr", stage_cost(wr, nt, R)))
        for nm, (t, i) in parts:
            total += t
            ideal += i
            if verbose:
                print(f"  R={R:2d} Ns={Ns:4d} {kind:5s} {nm}: {t:6d} wavefronts ({t / i:.2f}x ideal)")
    if verbose:
        print(f"L={L} plan={plan} axis={axis} B={B} LS={LS}: {total} wavefronts, {total / ideal:.3f}x ideal")
    return total / ideal


if __name__ == "__main__":
    L = int(sys.argv[1])
    plan = [int(x) for x in sys.argv[2:5] if x != "0"]
    axis = sys.argv[5] if len(sys.argv) > 5 else "row"
    B = int(sys.argv[6]) if len(sys.argv) > 6 else 1
    LS = int(sys.argv[7]) if len(sys.argv) > 7 else None
    analyze(L, plan, axis, B, LS)


def pad_search(L, plan, axis="row", B=1, LS=None):
    """Per inter-stage buffer, the skew period P (phys(i) = i + i // P, 0: none)
    that keeps every access affine in r and minimises wavefronts.
    Affine conditions: the writer (R, Ns) needs R | P (Ns = 1), P | Ns, or
    Ns R | P; the reader (T' = L / R') needs P | T'."""
    nst = len(plan)
    seq = []
    ns = 1
    for s, R in enumerate(plan):
        seq.append((R, ns))
        ns *= R
    rev = plan[::-1]
    ns = rev[0]
    for s in range(1, nst):
        seq.append((rev[s], ns))
        ns *= rev[s]
    # the mid stage (index nst-1) writes with the reversed plan's stage 0: (rev[0], 1)
    out = []
    for q in range(len(seq) - 1):
        Rw, Nsw = seq[q] if q != nst - 1 else (rev[0], 1)
        if q < nst - 1 and q > 0:
            Rw, Nsw = seq[q]
        if q == 0:
            Rw, Nsw = plan[0], 1
        Rr = seq[q + 1][0]
        Tr = L // Rr
        Tw = L // Rw
        cands = [0] + [P for P in range(2, L + 1) if Tr % P == 0 and
                       ((Nsw == 1 and P % Rw == 0) or (Nsw > 1 and (Nsw % P == 0 or P % (Nsw * Rw) == 0)))]
        best = None
        for P, c_ in [(P, c_) for P in cands for c_ in (range(1, 8) if P else [0])]:
            ph = (lambda i, P=P, c_=c_: i + c_ * (i // P)) if P else (lambda i: i)
            LSp = LS or (L + (c_ * (L // P) if P else 0))

            def dec(q_, T, nt):
                if q_ >= B * T:
                    return None
                return (q_ // T, q_ % T) if axis == "row" else (q_ % B, q_ // B)

            def wr(q_, r):
                d = dec(q_, Tw, 0)
                if d is None:
                    return None
                b, j = d
                k = j % Nsw
                return b * LSp + ph((j - k) * Rw + k + r * Nsw)

            def rd(q_, r):
                d = dec(q_, Tr, 0)
                if d is None:
                    return None
                return d[0] * LSp + ph(d[1] + r * Tr)

            ntw = ((B * Tw + 31) // 32) * 32
            ntr = ((B * Tr + 31) // 32) * 32
            tw, iw = stage_cost(wr, ntw, Rw)
            tr, ir = stage_cost(rd, ntr, Rr)
            c = (tw + tr) / (iw + ir)
            if best is None or c < best[1] - 1e-9:
                best = ((P, c_), c, tw / iw, tr / ir)
        out.append(best)
        print(f"  buffer after seq stage {q} (writer R={Rw} Ns={Nsw}, reader R={Rr}): best P={best[0]} -> {best[1]:.3f}x "
              f"(wr {best[2]:.2f}, rd {best[3]:.2f}); unpadded {[c for c in [0]] and ''}")
    return out


if __name__ == "__main__" and len(sys.argv) > 8 and sys.argv[8] == "pad":
    pad_search(int(sys.argv[1]), [int(x) for x in sys.argv[2:5] if x != "0"], sys.argv[5], int(sys.argv[6]),
               int(sys.argv[7]) or None)
