import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
data = np.load("tests/golden/small.npz"); meta = json.load(open("tests/golden/small.json"))
import paper_2503_06322_b200 as P
bad = []
for i, m in enumerate(meta):
    a = data[f"in{i}"]; vr = tuple(m["value_range"]) if m["value_range"] else None
    b = P.mgard_compress(a, m["eb_rel"], m["dict_size"], value_range=vr)
    ref = data[f"blob{i}"].tobytes()
    if b != ref:
        d = next((k for k in range(min(len(b), len(ref))) if b[k] != ref[k]), None)
        bad.append((i, m["shape"], m["dtype"], m["eb_rel"], vr, len(b), len(ref), d))
print("mismatches:", bad)
