"""CBC generating vectors -- bit-exact against the oracle's
exhaustive search; closed-form worst-case error known answers."""
import json
import math
import os

import numpy as np
import pytest

import paper_1808_06357_b200 as L
from oracle import pyoracle as O

CATALOG = json.load(open(os.path.join(os.path.dirname(L.__file__), "catalog.json")))


def test_wce_known_answers():
    # SPEC.md:123-125
    assert abs(L.wce_squared([1], 2) - math.pi ** 2 / 12) < 1e-15
    for n in (3, 7, 64, 1000):
        assert abs(L.wce_squared([1], n) - math.pi ** 2 / (3 * n * n)) < 1e-13 / n
    for d in (1, 2, 5):
        assert abs(L.wce_squared([3] * d, 1) - ((1 + 2 * math.pi ** 2 / 6) ** d - 1)) < 1e-12
    with pytest.raises(L.LattdseError) as e:
        L.wce_squared([1, 4], 16)
    assert e.value.name == "non_coprime_component"


def test_wce_matches_numpy_closed_form():
    rng = np.random.default_rng(3)
    for n in (97, 128, 1009):
        z = [int(x) for x in rng.integers(1, n, size=3) if math.gcd(int(x), n) == 1]
        k = np.arange(n)[:, None]
        x = (k * np.array(z)[None, :] % n) / n
        want = np.prod(1 + 2 * math.pi ** 2 * (x * x - x + 1 / 6), axis=1).mean() - 1
        assert abs(L.wce_squared(z, n) - want) < 1e-12


@pytest.mark.parametrize("n,d", [(32, 3), (64, 3), (2, 2), (101, 4), (257, 3), (1021, 3), (4099, 2)])
def test_cbc_equals_exhaustive_oracle(n, d):
    z, w = L.cbc_construct(n, d)
    zo, wo = O.cbc_exhaustive(n, d)
    assert z.tolist() == zo.tolist()
    # same criterion, independent omega tables: -1 + mean(...) cancels ~1, so absolute 1e-17
    assert np.allclose(w, wo, rtol=1e-12, atol=1e-17)
    assert z[0] == 1 and all(math.gcd(int(c), n) == 1 for c in z)
    for s in range(1, d):
        assert abs(L.wce_squared(z[: s + 1], n) - w[s]) <= 1e-12 * max(1.0, w[s])


def test_catalog_c0_exhaustive():
    cfg = CATALOG["C0"]
    zo, _ = O.cbc_exhaustive(cfg["n"], cfg["d"])
    assert zo.tolist() == cfg["z"]


def test_catalog_c3_recomputed():
    cfg = CATALOG["C3"]
    z, w = L.cbc_construct(cfg["n"], cfg["d"])
    assert z.tolist() == cfg["z"] and np.allclose(w, cfg["wce"], rtol=0, atol=0)


@pytest.mark.slow
def test_catalog_c1_recomputed():
    cfg = CATALOG["C1"]
    z, w = L.cbc_construct(cfg["n"], cfg["d"])
    assert z.tolist() == cfg["z"]


def test_config_lattices_validate_in_reference_goldens():
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lattice_ref.json")))
    hashes = {(tuple(c["moduli"]), tuple(map(tuple, c["gen"]))): c.get("hash") for c in gold["cases"]}
    for name, cfg in CATALOG.items():
        key = ((cfg["n"],), (tuple(cfg["z"]),))
        assert hashes[key] == "0x%016x" % L.Lattice.rank1(cfg["z"], cfg["n"]).hash()
