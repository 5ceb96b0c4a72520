"""Record the CBC generating vectors of the BASELINE rank-1 configs
(paper_1808_06357_b200/catalog.json). Produced by the product's cbc_construct
(prime-n extension of SPEC.md:128-137); tests/test_cbc.py re-derives them and
cross-checks the shortlist rule against the oracle's exhaustive search at
small n. Run: python tests/golden/make_cbc_configs.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
import paper_1808_06357_b200 as L  # noqa: E402

CONFIGS = {"C0": (4099, 2), "C1": (1048583, 6), "C3": (262147, 6)}
out = {}
for name, (n, d) in CONFIGS.items():
    z, w = L.cbc_construct(n, d)
    out[name] = {"n": n, "d": d, "z": [int(x) for x in z], "wce": [float(x) for x in w]}
    print(name, out[name]["z"])
with open(os.path.join(HERE, "..", "..", "paper_1808_06357_b200", "catalog.json"), "w") as f:
    json.dump(out, f, indent=1)
