"""The five BASELINE.json configurations as (lattice, problem, time grid).

Seed schedule: base seed 0x180806357 + config index;
one SplitMix64 stream draws a_1..a_d ~ U[0.5,1.5], b_1..b_{d-1} ~ U[0,0.5],
then (single wave function) c_1..c_d ~ U[c_lo,c_hi], p_1..p_d ~ U{-p..p};
ensemble member m draws (c, p) from a stream seeded with
SplitMix64(base ^ (m+1)).next(). v and z are shared by all members.

Generating vectors: paper_1808_06357_b200/catalog.json holds the prime-n CBC
vectors (recomputed and compared by tests/test_cbc.py). The reference has no
rank-r constructor, so config 2 uses a product rank-2
lattice built from the 8-D CBC vector z for n = 4096 (SPEC's power-of-two
CBC, odd candidates): Z = [(z1..z4, 0,0,0,0), (0,0,0,0, z5..z8)],
n = (4096, 4096). It is canonical (validated by Lattice.create: n2 | n1,
nonzero components odd, independent columns, 4096^2 distinct points) and its
minimal anti-aliasing set has max ||h||^2 = 96. The survey's example
Z = [(1,3,..,15), (0,1,3,..,13)] also validates, but its dual lattice has
short vectors: max ||h||^2 is already 163 at n = 128, so a norm table at
n = 4096 is out of reach.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import Lattice, cbc_construct, problem_draw

_HERE = os.path.dirname(os.path.abspath(__file__))
SEED_BASE = 0x180806357


@dataclass
class Config:
    name: str
    index: int
    d: int
    rank: int
    N: int                     # points (rank-2: n1*n2)
    moduli: tuple
    eps: float
    T: float
    m: int
    sigma: float
    batch: int
    c_range: tuple
    p_max: int
    gen: list = field(default_factory=list)  # rank columns of length d

    @property
    def dt(self) -> float:
        return self.T / self.m

    @property
    def seed(self) -> int:
        return SEED_BASE + self.index


def _catalog():
    with open(os.path.join(_HERE, "catalog.json")) as f:
        return json.load(f)


def _c(name, index, d, n, eps, T, m, sigma, batch=1, c_range=(0.4, 0.6), p_max=2, rank=1, moduli=None, gen=None):
    return Config(name, index, d, rank, int(np.prod(moduli)) if moduli else n, tuple(moduli or (n,)), eps, T, m,
                  sigma, batch, c_range, p_max, gen or [])


CONFIGS = {
    "C0": _c("C0", 0, 2, 4099, 0.1, 1.0, 256, 0.1),
    "C1": _c("C1", 1, 6, 1048583, 0.05, 1.0, 1024, 0.1),
    # product rank-2 lattice from the 8-D CBC vector for n = 4096 (see module doc)
    "C2": _c("C2", 2, 8, None, 0.05, 1.0, 512, 0.08, rank=2, moduli=(4096, 4096),
             gen=[[1, 1557, 1741, 1031, 0, 0, 0, 0], [0, 0, 0, 0, 363, 1705, 1349, 1667]]),
    "C3": _c("C3", 3, 6, 262147, 0.05, 0.5, 512, 0.1, batch=512, c_range=(0.3, 0.7), p_max=3),
    "C4": _c("C4", 4, 20, 1073741827, 0.02, 0.1, 64, 0.15),
    # config 4's shape at reduced N: d = 20, N = smallest
    # prime >= 2^24; oracle-checkable, and the three-level layout's test case
    "C4r": _c("C4r", 5, 20, 16777259, 0.02, 0.1, 64, 0.15),
}


def generating_vector(cfg: Config, recompute: bool = False):
    cat = _catalog()
    if not recompute and cfg.name in cat:
        return cat[cfg.name]["z"]
    z, _ = cbc_construct(cfg.N, cfg.d)
    return [int(x) for x in z]


def lattice(cfg: Config, recompute: bool = False) -> Lattice:
    if cfg.rank == 2:
        return Lattice.create(cfg.d, 2, cfg.gen, cfg.moduli)
    return Lattice.rank1(generating_vector(cfg, recompute), cfg.N)


def problem(cfg: Config, batch: int | None = None):
    """(a, b, c[batch,d], p[batch,d]) from the seed schedule."""
    batch = cfg.batch if batch is None else batch
    a, b, c, p = problem_draw(cfg.seed, cfg.d, cfg.batch, cfg.c_range[0], cfg.c_range[1], cfg.p_max)
    return a, b, c[:batch], p[:batch]


def small_rank1(d: int, n: int, eps=0.1, sigma=0.1, seed=7, batch=1, c_range=(0.4, 0.6), p_max=2):
    """Test-size rank-1 problem: CBC lattice + seeded families."""
    z, _ = cbc_construct(n, d)
    lat = Lattice.rank1(z, n)
    a, b, c, p = problem_draw(seed, d, batch, c_range[0], c_range[1], p_max)
    return lat, a, b, c, p


def rank2_product(n1: int, n2: int, d: int):
    """Product rank-2 lattice as used by config 2: CBC vector z for n1 in d
    dimensions, Z = [(z_1..z_h, 0..0), (0..0, z_{h+1}..z_d) mod n2], h = d//2."""
    z, _ = cbc_construct(n1, d)
    h = d // 2
    c1 = [int(x) for x in z[:h]] + [0] * (d - h)
    c2 = [0] * h + [int(x) % n2 for x in z[h:]]
    return Lattice.create(d, 2, [c1, c2], [n1, n2])


def shard_members(batch: int, rank: int, world: int):
    """Contiguous ensemble shard of `rank` (config 3 batch sharding, SURVEY.md
    §8(e)): returns (first member, count); shards differ in size by <= 1."""
    base, extra = divmod(batch, world)
    m0 = rank * base + min(rank, extra)
    return m0, base + (1 if rank < extra else 0)
