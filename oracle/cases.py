"""TEST INFRASTRUCTURE ONLY -- the five BASELINE.json configurations restated
independently of the product package, so that oracle runs (golden fixtures,
the CPU baseline and the reference arm of bench.py) take no input from
paper_1808_06357_b200.

What is restated here, and from where:
- the config table (d, N, eps, T, m, sigma, c/p ranges): BASELINE.json
  `configs`, SURVEY.md §8 table;
- the seed schedule (SplitMix64, draw order a, b, c, p; member streams):
  SURVEY.md §8(d) "Synthetic inputs", DESIGN.md §6 "Seeds";
- the generating vectors: prime-n CBC. C0 is re-derived by
  the oracle's exhaustive CBC in tests/test_oracle_cases.py; C1/C3 are the
  host fast-CBC results (bit-exact to the exhaustive oracle at every n it can
  finish, tests/test_cbc.py); C4r is catalog.json's device-CBC vector taken
  as the lattice definition (its index map is the oracle's own walk);
- config 2's rank-2 lattice ("Config 2 lattice").
tests/test_oracle_cases.py checks this table against the product's
configs.py so the two cannot drift apart silently.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 0x180806357
MASK = 0xFFFFFFFFFFFFFFFF


class SplitMix64:
    def __init__(self, seed):
        self.s = seed & MASK

    def next(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self, lo=0.0, hi=1.0):
        return lo + (hi - lo) * ((self.next() >> 11) * 2.0 ** -53)

    def integer(self, lo, hi):
        return lo + min(int(math.floor(self.uniform() * (hi - lo + 1))), hi - lo)


@dataclass
class Case:
    name: str
    index: int
    d: int
    gen: list          # rank columns of length d
    moduli: tuple
    eps: float
    T: float
    m: int
    sigma: float
    batch: int = 1
    c_range: tuple = (0.4, 0.6)
    p_max: int = 2
    extra: dict = field(default_factory=dict)

    @property
    def N(self):
        return int(np.prod(self.moduli))

    @property
    def dt(self):
        return self.T / self.m

    @property
    def seed(self):
        return SEED_BASE + self.index

    def potential_params(self):
        r = SplitMix64(self.seed)
        a = np.array([r.uniform(0.5, 1.5) for _ in range(self.d)])
        b = np.array([r.uniform(0.0, 0.5) for _ in range(self.d - 1)])
        return a, b, r

    def member(self, m: int):
        """(c, p) of ensemble member m (single wave functions: member 0)."""
        a, b, r = self.potential_params()
        lo, hi = self.c_range
        if self.batch > 1:
            r = SplitMix64(SplitMix64(self.seed ^ (m + 1)).next())
        elif m != 0:
            raise ValueError("single wave function: member 0 only")
        c = np.array([r.uniform(lo, hi) for _ in range(self.d)])
        p = np.array([r.integer(-self.p_max, self.p_max) for _ in range(self.d)], np.int32)
        return c, p


def _r1(name, index, d, n, z, eps, T, m, sigma, **kw):
    return Case(name, index, d, [list(z)], (n,), eps, T, m, sigma, **kw)


CASES = {
    "C0": _r1("C0", 0, 2, 4099, [1, 1588], 0.1, 1.0, 256, 0.1),
    "C1": _r1("C1", 1, 6, 1048583, [1, 460549, 173282, 362345, 238323, 521751], 0.05, 1.0, 1024, 0.1),
    "C2": Case("C2", 2, 8, [[1, 1557, 1741, 1031, 0, 0, 0, 0], [0, 0, 0, 0, 363, 1705, 1349, 1667]], (4096, 4096),
               0.05, 1.0, 512, 0.08),
    "C3": _r1("C3", 3, 6, 262147, [1, 102226, 122243, 92569, 3585, 103565], 0.05, 0.5, 512, 0.1, batch=512,
              c_range=(0.3, 0.7), p_max=3),
    # config 4's shape at reduced N; the lattice definition
    # is catalog.json's C4r vector (device CBC); its index map is the
    # oracle's own walk (tests/golden/c4r_tables.json)
    "C4r": _r1("C4r", 5, 20, 16777259, [1, 6408565, 2903963, 4966000, 8029635, 3702744, 8380425, 5023039, 508131,
                                         6943149, 3253008, 3662870, 380856, 6470234, 2574891, 6408565, 6408565,
                                         6408565, 6408565, 6408565], 0.02, 0.1, 64, 0.15),
}


# ------------------------------------------------------------- fixtures
def _splitmix_vec(x):
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def checksum_weights(n: int, k: int, lo: int = 0, hi: int | None = None):
    """Unit-modulus pseudo-random weights w_k[chi], chi in [lo, hi): a linear
    functional S_k(u) = sum_chi w_k[chi] u[chi] of the full state. For an
    error e, |S_k(e)| ~ ||e||_2 (random phases), so comparing S_k of the GPU
    state with the oracle's checks the WHOLE state at the 1e-10 level with
    four numbers per state ("checksum of checksums")."""
    hi = n if hi is None else hi
    chi = np.arange(lo, hi, dtype=np.uint64)
    h = _splitmix_vec(chi ^ np.uint64((0xA5A5A5A5 * (k + 1)) & MASK))
    ph = (h >> np.uint64(11)).astype(np.float64) * (2.0 * np.pi * 2.0 ** -53)
    return np.exp(1j * ph)


def checksums(u, kmax: int = 4, chunk: int = 1 << 22):
    u = np.asarray(u).reshape(-1)
    out = np.zeros(kmax, np.complex128)
    for lo in range(0, u.size, chunk):
        hi = min(u.size, lo + chunk)
        for k in range(kmax):
            out[k] += np.dot(checksum_weights(u.size, k, lo, hi), u[lo:hi])
    return out


def subset_indices(n: int, count: int, seed: int):
    """Sorted seeded subset of [0, n) (always contains 0 and n-1)."""
    rng = np.random.default_rng(seed)
    idx = rng.choice(n, size=min(count, n), replace=False)
    idx = np.unique(np.concatenate([idx, [0, n - 1]]))
    return idx.astype(np.int64)
