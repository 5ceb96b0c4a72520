"""Independent index map for config 4r (d = 20, N = 16777259): the ORACLE's
literal shell walk (oracle.cpp orc_aaset) builds the norm table
of the C4r lattice, and its sha256 is committed (tests/golden/c4r_tables.json).
tests/test_gpu_config4.py then requires the product's device meet-in-the-
middle walk to hash identically before the oracle is fed that table at test
time (the walk itself is too slow for a test run). The generating vector is
the lattice definition (catalog.json C4r); the host fast CBC's result for the
same (n, d) is recorded next to it when tools/c4r_host_cbc.py finished.

    python tests/golden/make_c4r_golden.py [host_cbc.json]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402

cat = json.load(open(os.path.join(ROOT, "paper_1808_06357_b200", "catalog.json")))["C4r"]
z, n = [int(x) for x in cat["z"]], int(cat["n"])
t0 = time.time()
norm2, _ = po.aaset([z], [n], with_vectors=False)
out = {"n": n, "d": len(z), "z": z, "z_source": cat.get("construction"),
       "norm2_sha256": hashlib.sha256(np.ascontiguousarray(norm2, np.uint32).tobytes()).hexdigest(),
       "max_norm2": int(norm2.max()), "oracle_walk_seconds": round(time.time() - t0, 1),
       "shell_counts": np.bincount(norm2).tolist()}
if len(sys.argv) > 1 and os.path.exists(sys.argv[1]) and os.path.getsize(sys.argv[1]) > 0:
    h = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    out["host_fast_cbc"] = {"z": h["z"], "wce": h["wce"], "seconds": h["seconds"], "equals_catalog": h["z"] == z}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "c4r_tables.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "shell_counts"}))
