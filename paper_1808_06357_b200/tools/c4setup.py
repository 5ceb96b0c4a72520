# Generates the config-4 generating vectors with the device CBC (catalog.json
# entries C4, C4r) and times the device anti-aliasing norm build. GPU box:
#   python paper_1808_06357_b200/tools/c4setup.py  -> gpurun_out/c4setup.json
import json, sys, time
import numpy as np
import paper_1808_06357_b200 as L
out = {}
for name, n in (("C4r", 16777259), ("C4", 1073741827)):
    t = time.time()
    z, w = L.cbc_construct_device(n, 20)
    out[name] = {"n": n, "d": 20, "z": [int(x) for x in z], "wce": [float(x) for x in w], "cbc_s": time.time() - t}
    print(name, "cbc", out[name]["cbc_s"], out[name]["z"], flush=True)
    lat = L.Lattice.rank1(out[name]["z"], n)
    t = time.time()
    if name == "C4r":
        norm2, mx = L.aaset_norms_device(lat)
        out[name]["max_norm2"] = int(mx)
        out[name]["norm_hist"] = np.bincount(norm2).tolist()
    else:
        import ctypes as C
        mx = C.c_uint32()
        L._ck(L._lib.lattdse_aaset_norms_device(lat.handle, 0, C.c_double(-1.0), None, C.byref(mx)))
        out[name]["max_norm2"] = int(mx.value)
    out[name]["aaset_s"] = time.time() - t
    print(name, "aaset", out[name]["aaset_s"], out[name]["max_norm2"], flush=True)
import os
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/c4setup.json", "w"), indent=1)
