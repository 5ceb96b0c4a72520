"""Snapshot write/read (include/lattdse/snapshot.hpp):
round trip, sidecar contents, and the error codes for a foreign lattice,
a truncated data file and a missing sidecar. Host-only (no GPU)."""
import json

import numpy as np
import pytest

import paper_1808_06357_b200 as L


def test_round_trip(tmp_path):
    lat = L.Lattice.rank1([1, 34], 55)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 55)) + 1j * rng.standard_normal((3, 55))
    path = str(tmp_path / "u.c128")
    L.snapshot_write(lat, path, x, space=L.COEFFICIENTS, step=17, time=0.25, dt=1 / 64)
    raw = np.fromfile(path, dtype="<c16")
    assert raw.size == 3 * 55 and np.array_equal(raw.reshape(3, 55), x)
    side = json.load(open(path + ".json"))
    assert side["length"] == 55 and side["members"] == 3 and side["ordering"] == "chi"
    assert side["lattice_hash"] == f"0x{lat.hash():016x}"
    assert L.Lattice.from_json(json.dumps(side["lattice"])) == lat
    y, meta = L.snapshot_read(lat, path)
    assert np.array_equal(y, x)
    assert meta == {"members": 3, "space": L.COEFFICIENTS, "step": 17, "time": 0.25, "dt": 1 / 64}


def test_errors(tmp_path):
    lat = L.Lattice.rank1([1, 34], 55)
    other = L.Lattice.rank1([1, 21], 55)
    path = str(tmp_path / "u.c128")
    L.snapshot_write(lat, path, np.ones(55, complex))
    with pytest.raises(L.LattdseError) as e:
        L.snapshot_read(other, path)
    assert e.value.name == "config_error"  # lattice hash mismatch
    with open(path, "r+b") as f:
        f.truncate(100)
    with pytest.raises(L.LattdseError) as e:
        L.snapshot_read(lat, path)
    assert e.value.name == "io_error"  # truncated
    with pytest.raises(L.LattdseError) as e:
        L.snapshot_read(lat, str(tmp_path / "missing.c128"))
    assert e.value.name == "io_error"
