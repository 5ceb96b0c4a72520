"""lattice-core parity with the REFERENCE implementation (CPU).

tests/golden/lattice_ref.json was produced by the reference's own
lattice.cpp (compiled from /root/reference by oracle/build_ref.sh, generator
tests/golden/make_lattice_golden.py). The product's fresh Lattice must return
the same error codes, hashes, JSON, points and residues. Plus the SPEC.md
examples and properties.
"""
import json
import os

import numpy as np
import pytest

import paper_1808_06357_b200 as L

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lattice_ref.json")))


def make(case):
    return L.Lattice.create(case["dim"], case["rank"], case["gen"], case["moduli"])


@pytest.mark.parametrize("idx", range(len(GOLD["cases"])))
def test_reference_golden(idx):
    case = GOLD["cases"][idx]
    if case["code"] != 0:
        with pytest.raises(L.LattdseError) as e:
            make(case)
        assert e.value.code + 1 == case["code"], e.value
        return
    lat = make(case)
    assert "0x%016x" % lat.hash() == case["hash"]
    assert lat.to_json() == case["json"]
    assert lat.denom() == case["denom"]
    if "points" in case:
        assert np.array_equal(lat.point_numerators(), np.array(case["points"]))
    if "point_rows" in case:
        pts = lat.point_numerators()
        for k, row in case["point_rows"].items():
            assert pts[int(k)].tolist() == row
        assert pts.sum(axis=0).tolist() == case["points_sum"]
    for r in case["residues"]:
        assert lat.residue(r["h"]).tolist() == r["xi"]
        assert lat.flat_residue(r["h"]) == r["flat"]
        assert lat.in_dual(r["h"]) == bool(r["dual"])


def test_from_json_codes():
    for case in GOLD["from_json"]:
        if case["code"] == 0:
            lat = L.Lattice.from_json(case["text"])
            assert lat.to_json() == '{"Z":[[1,34]],"d":2,"n":[55],"r":1}'
        else:
            with pytest.raises(L.LattdseError) as e:
                L.Lattice.from_json(case["text"])
            assert e.value.code + 1 == case["code"]


def test_rank1_fixed_and_equal_to_create():
    # the reference's rank1() throws under GCC (lattice.cpp:237-239)
    assert GOLD["rank1_reference_bug"]["code"] == 1
    a = L.Lattice.rank1([1, 34], 55)
    b = L.Lattice.create(2, 1, [[1, 34]], [55])
    assert a == b and a.hash() == b.hash() == 0xC52FC32F65226F72


def test_spec_examples():
    # SPEC.md:55-57
    assert (L.Lattice.rank1([1], 4).point_coords()[:, 0] == [0, 0.25, 0.5, 0.75]).all()
    assert L.Lattice.rank1([1, 34], 55).point_numerators()[1].tolist() == [1, 34]
    g = L.Lattice.grid([2, 2])
    assert sorted(map(tuple, g.point_coords().tolist())) == [(0, 0), (0, 0.5), (0.5, 0), (0.5, 0.5)]
    # SPEC.md:65-77
    lat = L.Lattice.rank1([1, 34], 55)
    assert lat.in_dual([0, 0]) and lat.in_dual([55, 0]) and lat.in_dual([21, 1]) and not lat.in_dual([1, 0])
    assert lat.residue([1, 0]).tolist() == [1] and lat.residue([0, 2]).tolist() == [13]
    # SPEC.md:47
    L.Lattice.create(2, 1, [[2, 34]], [55])
    with pytest.raises(L.LattdseError) as e:
        L.Lattice.create(2, 1, [[5, 34]], [55])
    assert e.value.name == "non_coprime_component"
    assert lat.point_index(7).tolist() == [7]
    assert L.Lattice.grid([4, 2]).point_index(5).tolist() == [2, 1]


@pytest.mark.parametrize("seed", range(6))
def test_character_property_and_additivity(seed):
    # (1/n) sum_p exp(2 pi i h.p) = [h in dual]; residue additive;
    # points distinct
    rng = np.random.default_rng(seed)
    if seed % 2:
        n = int(rng.choice([16, 64, 97, 128, 255]))
        d = int(rng.integers(1, 4))
        while True:
            z = rng.integers(1, n, size=d)
            if all(np.gcd(int(x), n) == 1 for x in z):
                break
        lat = L.Lattice.rank1(z, n)
    else:
        lat = L.Lattice.grid([8, 4] if seed == 0 else [6, 3, 3])
    d = lat.dim()
    pts = lat.point_coords()
    assert len({tuple(p) for p in lat.point_numerators().tolist()}) == lat.n_total()
    for _ in range(40):
        h = rng.integers(-8, 9, size=d)
        ch = np.exp(2j * np.pi * (pts @ h)).mean()
        assert abs(ch - (1.0 if lat.in_dual(h) else 0.0)) < 1e-10
        h2 = rng.integers(-8, 9, size=d)
        n = lat.moduli()
        assert ((lat.residue(h) + lat.residue(h2)) % n == lat.residue(h + h2)).all()
        assert (lat.residue(h) == 0).all() == lat.in_dual(h)


def test_errors_and_validation_order():
    with pytest.raises(L.LattdseError) as e:
        L.Lattice.create(2, 2, [[1, 0], [0, 1]], [4, 8])
    assert e.value.name == "non_divisible_moduli"
    with pytest.raises(L.LattdseError) as e:
        L.Lattice.create(3, 2, [[1, 3, 5], [3, 9, 15]], [4, 4])
    assert e.value.name == "rank_deficient"
    with pytest.raises(L.LattdseError) as e:
        L.Lattice.create(2, 2, [[1, 1], [1, 3]], [4, 4])
    assert e.value.name == "point_count_mismatch"
    with pytest.raises(L.LattdseError) as e:
        L.Lattice.rank1([1, 3], 1 << 41)
    assert e.value.name == "overflow_risk"
