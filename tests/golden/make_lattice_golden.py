"""Generate tests/golden/lattice_ref.json from the REFERENCE's own lattice-core.

Runs oracle/build_ref.sh (compiles /root/reference/proj/src/core/lattice.cpp in
place into oracle/_ref/libref_lattice.so) and records, for a fixed list of
lattices, what the reference returns: error code, FNV-1a hash, to_json,
denominator, point numerators and residue / in_dual answers for fixed h.
Run in the build container (the reference is not on the GPU boxes):

    python tests/golden/make_lattice_golden.py
"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

# generating vectors of the BASELINE rank-1 configs come from our CBC (the
# reference has no constructor for prime n); the reference then validates and
# hashes them.
CONFIG_Z = json.load(open(os.path.join(ROOT, "paper_1808_06357_b200", "catalog.json")))


def load_ref():
    subprocess.run([os.path.join(ROOT, "oracle", "build_ref.sh")], check=True)
    lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_lattice.so"))
    lib.ref_lattice_hash.restype = C.c_uint64
    lib.ref_lattice_denom.restype = C.c_int64
    return lib


def case(lib, dim, rank, gen, moduli, residue_hs=(), all_points_max=5000, point_rows=()):
    g = np.ascontiguousarray(np.asarray(gen, np.int64).reshape(-1))
    n = np.ascontiguousarray(np.asarray(moduli, np.int64).reshape(-1))
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib.ref_lattice_create(dim, rank, g.ctypes.data_as(C.POINTER(C.c_int64)),
                                n.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(h), err, 512)
    out = {"dim": dim, "rank": rank, "gen": np.asarray(gen).tolist(), "moduli": list(map(int, moduli)),
           "code": rc}
    if rc != 0:
        out["message"] = err.value.decode()
        return out
    out["hash"] = "0x%016x" % lib.ref_lattice_hash(h)
    out["denom"] = lib.ref_lattice_denom(h)
    buf = C.create_string_buffer(1 << 16)
    lib.ref_lattice_to_json(h, buf, 1 << 16)
    out["json"] = buf.value.decode()
    ntot = int(np.prod(n))
    if ntot <= all_points_max:
        pts = np.zeros((ntot, dim), np.int64)
        lib.ref_lattice_points(h, pts.ctypes.data_as(C.POINTER(C.c_int64)))
        out["points"] = pts.tolist()
    elif point_rows and ntot * dim <= 500_000_000:  # the reference enumerates every point
        pts = np.zeros((ntot, dim), np.int64)
        lib.ref_lattice_points(h, pts.ctypes.data_as(C.POINTER(C.c_int64)))
        out["point_rows"] = {str(k): pts[k].tolist() for k in point_rows}
        out["points_sum"] = [int(x) for x in pts.sum(axis=0)]
    res = []
    for hv in residue_hs:
        hv = np.ascontiguousarray(np.asarray(hv, np.int64))
        xi = np.zeros(rank, np.int64)
        flat = C.c_int64()
        dual = C.c_int()
        lib.ref_lattice_residue(h, hv.ctypes.data_as(C.POINTER(C.c_int64)), xi.ctypes.data_as(C.POINTER(C.c_int64)),
                                C.byref(flat), C.byref(dual))
        res.append({"h": hv.tolist(), "xi": xi.tolist(), "flat": flat.value, "dual": dual.value})
    out["residues"] = res
    lib.ref_lattice_destroy(h)
    return out


def main():
    lib = load_ref()
    rng = np.random.default_rng(1808_06357)
    cases = []
    # SPEC.md:44-77 examples
    cases.append(case(lib, 2, 1, [[1, 34]], [55], [[0, 0], [1, 0], [0, 2], [55, 0], [21, 1], [-3, 7], [100, -41]]))
    cases.append(case(lib, 2, 1, [[2, 34]], [55], [[1, 1], [3, -2]]))
    cases.append(case(lib, 2, 1, [[5, 34]], [55]))                       # non_coprime_component
    cases.append(case(lib, 1, 1, [[1]], [4], [[1], [5], [-1]]))
    cases.append(case(lib, 2, 2, [[1, 0], [0, 1]], [4, 4], [[1, 2], [-1, 5], [4, 4]]))
    cases.append(case(lib, 2, 2, [[1, 0], [0, 1]], [2, 2], [[1, 1]]))
    cases.append(case(lib, 2, 2, [[1, 0], [0, 1]], [4, 8]))               # non_divisible_moduli
    cases.append(case(lib, 3, 2, [[1, 2, 3], [2, 4, 6]], [4, 4]))         # non_coprime before rank check
    cases.append(case(lib, 3, 2, [[1, 3, 5], [3, 9, 15]], [4, 4]))        # rank_deficient
    cases.append(case(lib, 2, 2, [[1, 1], [1, 3]], [4, 4]))               # point_count_mismatch
    cases.append(case(lib, 2, 1, [[1, 3]], [1 << 41]))                    # overflow_risk (lcm)
    cases.append(case(lib, 2, 1, [[1, (1 << 30) + 1]], [1 << 33]))        # overflow_risk (lcm*z)
    cases.append(case(lib, 0, 1, [[]], [5]))                              # invalid_argument
    cases.append(case(lib, 2, 1, [[1, 3]], [0]))                          # invalid_argument (modulus)
    cases.append(case(lib, 3, 3, np.eye(3, dtype=int).tolist(), [6, 3, 3], [[1, 2, 3], [7, -1, 4]]))
    cases.append(case(lib, 4, 2, [[1, 3, 5, 7], [0, 1, 3, 5]], [8, 4], [[1, 2, 3, 4], [-2, 0, 1, 9]]))
    cases.append(case(lib, 3, 1, [[1, 0, 7]], [16], [[1, 1, 1], [0, 3, -2]]))   # zero component allowed
    cases.append(case(lib, 3, 2, [[2, 0, 0], [0, 1, 0]], [4, 4]))         # non_coprime (2 vs 4)
    # the survey's example rank-2 generator (validates; not used: poor aaset)
    z2 = [[1, 3, 5, 7, 9, 11, 13, 15], [0, 1, 3, 5, 7, 9, 11, 13]]
    hs = rng.integers(-9, 10, size=(16, 8)).tolist()
    cases.append(case(lib, 8, 2, z2, [4096, 4096], hs, point_rows=[0, 1, 4095, 4096, 4097, 16777215]))
    # the rank-2 lattice of config 2 (product of the 8-D CBC vector halves)
    z2 = [[1, 1557, 1741, 1031, 0, 0, 0, 0], [0, 0, 0, 0, 363, 1705, 1349, 1667]]
    hs = rng.integers(-9, 10, size=(16, 8)).tolist()
    cases.append(case(lib, 8, 2, z2, [4096, 4096], hs, point_rows=[0, 1, 4095, 4096, 4097, 16777215]))
    # the rank-1 config lattices with our CBC vectors
    for name, cfg in CONFIG_Z.items():
        d = len(cfg["z"])
        hs = rng.integers(-12, 13, size=(12, d)).tolist()
        rows = [0, 1, 2, 3, cfg["n"] - 1]
        cases.append(case(lib, d, 1, [cfg["z"]], [cfg["n"]], hs, all_points_max=5000, point_rows=rows))
    # random small valid/invalid rank-1 lattices
    for _ in range(12):
        n = int(rng.integers(2, 300))
        d = int(rng.integers(1, 5))
        z = rng.integers(-n, 2 * n, size=d).tolist()
        hs = rng.integers(-20, 21, size=(6, d)).tolist()
        cases.append(case(lib, d, 1, [z], [n], hs))
    # from_json behaviour
    js = []
    for text in ['{"d":2,"r":1,"Z":[[1,34]],"n":[55]}', '{"d":2,"r":1,"Z":[[1,34]]}', "{not json",
                 '{"d":2,"r":1,"Z":[[1,"a"]],"n":[55]}']:
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib.ref_lattice_from_json(text.encode(), C.byref(h), err, 512)
        js.append({"text": text, "code": rc})
        if rc == 0:
            lib.ref_lattice_destroy(h)
    # the reference's rank1() evaluation-order bug (lattice.cpp:237-239)
    z = np.array([1, 34], np.int64)
    err = C.create_string_buffer(512)
    rc1 = lib.ref_lattice_rank1_raw(z.ctypes.data_as(C.POINTER(C.c_int64)), 2, 55, err, 512)
    out = {"generator": "tests/golden/make_lattice_golden.py (reference lattice.cpp compiled by oracle/build_ref.sh)",
           "cases": cases, "from_json": js, "rank1_reference_bug": {"code": rc1, "message": err.value.decode()}}
    with open(os.path.join(HERE, "lattice_ref.json"), "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
