"""Generate the full-run parity fixtures (tests/golden/run_<case>.npz) with
the CPU ORACLE (oracle/oracle.cpp, literal SPEC.md:336-344 Strang step, its
own FFT and its own shell-walk anti-aliasing set). No input comes from the
product package: lattices, seeds and parameters are oracle/cases.py.

Per case and member the fixture holds
  idx          seeded subset of coefficient indices (chi order)
  u1, um       coefficients after 1 and after m Strang steps, at idx
  cs1, csm     checksums(S_0..S_3) of the FULL coefficient vector (oracle/cases.py)
  nrm1/nrmm    ||u|| after 1 / m steps, energy_m
  norm2_sha    sha256 of the oracle's uint32 norm table (the GPU test compares
               the product's table hash with it: an independent index map)
Run:  python tests/golden/make_run_fixtures.py C3 C1 C2   (~80 min on 8 cores)
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402
from oracle.cases import CASES, checksums, subset_indices  # noqa: E402

SUBSET = {"C0": 1 << 12, "C1": 1 << 17, "C2": 1 << 17, "C3": 1 << 16}
MEMBERS = {"C3": [0, 255, 511]}


def run(name):
    cs = CASES[name]
    t0 = time.time()
    norm2, _ = po.aaset(cs.gen, cs.moduli, with_vectors=False)
    a, b, _ = cs.potential_params()
    orc = po.Oracle(cs.gen, cs.moduli, norm2, cs.eps, a, b)
    orc.set_dt(cs.dt)
    idx = subset_indices(cs.N, SUBSET[name], seed=cs.seed)
    out = {"idx": idx, "norm2_sha": np.frombuffer(hashlib.sha256(norm2.tobytes()).digest(), np.uint8),
           "m": np.int64(cs.m), "N": np.int64(cs.N)}
    members = MEMBERS.get(name, [0])
    out["members"] = np.array(members, np.int64)
    for mi, mem in enumerate(members):
        c, p = cs.member(mem)
        u = orc.analyze(orc.initial_samples(c, p, cs.sigma))
        u = orc.steps(u, 1)
        out[f"u1_{mi}"] = u[idx]
        out[f"cs1_{mi}"] = checksums(u)
        out[f"nrm1_{mi}"] = np.float64(orc.l2_norm(u))
        done = 1
        while done < cs.m:
            k = min(64, cs.m - done)
            u = orc.steps(u, k)
            done += k
            print(f"{name} member {mem}: {done}/{cs.m} steps, {time.time() - t0:.0f} s", flush=True)
        out[f"um_{mi}"] = u[idx]
        out[f"csm_{mi}"] = checksums(u)
        out[f"nrmm_{mi}"] = np.float64(orc.l2_norm(u))
        out[f"enm_{mi}"] = np.float64(orc.energy(u))
    path = os.path.join(ROOT, "tests", "golden", f"run_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path} in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["C0", "C3", "C1", "C2"]:
        run(nm)
