"""Record the CBC generating vectors of the BASELINE rank-1 configs
(paper_1808_06357_b200/catalog.json). Produced by the product's cbc_construct
(prime-n extension of SPEC.md:128-137); tests/test_cbc.py re-derives them and
cross-checks the shortlist rule against the oracle's exhaustive search at
small n. Run: python paper_1808_06357_b200/tools/make_catalog.py
Entries built on the device (C4, C4r: tools/c4setup.py on a GPU box) are kept.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
import paper_1808_06357_b200 as L  # noqa: E402

CONFIGS = {"C0": (4099, 2), "C1": (1048583, 6), "C3": (262147, 6)}
PATH = os.path.join(HERE, "..", "catalog.json")
with open(PATH) as f:
    out = json.load(f)
for name, (n, d) in CONFIGS.items():
    z, w = L.cbc_construct(n, d)
    out[name] = {"n": n, "d": d, "z": [int(x) for x in z], "wce": [float(x) for x in w],
                 "construction": "host (cbc_construct)"}
    print(name, out[name]["z"])
with open(PATH, "w") as f:
    json.dump(out, f, indent=1)
