"""Minimal-l2 anti-aliasing set: the product's parallel
(norm, lex)-minimum construction vs the oracle's literal shell walk, bit-exact
(norm table and h table), plus SPEC's examples and properties."""
import numpy as np
import pytest

import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
from oracle import pyoracle as O


def both(gen, moduli):
    gen = np.asarray(gen)
    lat = L.Lattice.create(gen.shape[1], gen.shape[0], gen, moduli)
    n2, h, mx = L.aaset_build(lat)
    on2, oh = O.aaset(gen, moduli)
    return lat, n2, h, mx, on2, oh


def test_fig1_lattice():
    # card 55, h(0) = 0, h(1) = (1,0)
    lat, n2, h, mx, on2, oh = both([[1, 34]], [55])
    assert len(n2) == 55 and h[0].tolist() == [0, 0] and h[1].tolist() == [1, 0]
    assert np.array_equal(n2, on2) and np.array_equal(h, oh)
    # residue bijectivity and minimality by brute force over |h|_inf <= 8
    assert sorted(lat.flat_residue(x) for x in h) == list(range(55))
    best = {}
    for a in range(-8, 9):
        for b in range(-8, 9):
            r = lat.flat_residue([a, b])
            best[r] = min(best.get(r, 10 ** 9), a * a + b * b)
    assert all(best[r] == n2[r] for r in range(55))


def test_grid_4x4_centered():
    # every class represented once, minimal norm, lexicographic ties
    lat, n2, h, mx, on2, oh = both([[1, 0], [0, 1]], [4, 4])
    assert np.array_equal(h, oh)
    assert set(map(tuple, h.tolist())) <= {(a, b) for a in range(-2, 3) for b in range(-2, 3)}
    assert h[lat.flat_residue([2, 0])].tolist() == [-2, 0]  # (-2,0) < (2,0)


@pytest.mark.parametrize("seed", range(10))
def test_random_small_lattices_match_oracle(seed):
    # acceptance 3: exhaustive minimality on random n <= 2^9, d <= 4
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 512))
    d = int(rng.integers(1, 5))
    while True:
        z = rng.integers(1, n, size=d)
        if all(np.gcd(int(x), n) == 1 for x in z):
            break
    lat, n2, h, mx, on2, oh = both([z.tolist()], [n])
    assert np.array_equal(n2, on2) and np.array_equal(h, oh)
    assert mx == n2.max()
    # anti-aliasing (Definition 2.2): no two members differ by a dual vector
    res = [lat.flat_residue(x) for x in h]
    assert len(set(res)) == n


def test_rank2_product_lattice():
    lat = configs.rank2_product(64, 32, 4)
    gen, moduli = lat.generators()
    n2, h, mx = L.aaset_build(lat)
    on2, oh = O.aaset(gen, moduli)
    assert np.array_equal(n2, on2) and np.array_equal(h, oh)


@pytest.mark.parametrize("name", ["C0", "C3", "C1"])
def test_config_norm_tables(name):
    cfg = configs.CONFIGS[name]
    lat = configs.lattice(cfg)
    n2, h, mx = L.aaset_build(lat)
    gen, moduli = lat.generators()
    on2, oh = O.aaset(gen, moduli)
    assert np.array_equal(n2, on2) and np.array_equal(h, oh)


@pytest.mark.slow
def test_config2_norm_table():
    cfg = configs.CONFIGS["C2"]
    lat = configs.lattice(cfg)
    n2, _, mx = L.aaset_build(lat, with_vectors=False)
    gen, moduli = lat.generators()
    on2, _ = O.aaset(gen, moduli, with_vectors=False)
    assert mx == 96 and np.array_equal(n2, on2)


def test_radius_exhausted():
    lat = L.Lattice.rank1([1, 34], 55)
    with pytest.raises(L.LattdseError) as e:
        L.aaset_build(lat, cap_radius=2.0)
    assert e.value.name == "radius_exhausted"
