"""Host fast CBC (csrc/host/cbc.cpp: Rader-FFT shortlist re-scored with the
exact long-double criterion) for config 4r, N = 16777259, d = 20 -- an
independent check of the device construction that produced catalog.json's
C4r vector. Prints the vector, per-component criteria and the time.

    python paper_1808_06357_b200/tools/c4r_host_cbc.py [n] [d]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
import paper_1808_06357_b200 as L  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16777259
d = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
z, w = L.cbc_construct(n, d)
print(json.dumps({"n": n, "d": d, "z": [int(x) for x in z], "wce": [float(x) for x in w],
                  "seconds": time.time() - t0}), flush=True)
