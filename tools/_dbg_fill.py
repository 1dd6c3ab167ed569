import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import _lib
orig = _lib.new_bytes
def filled(n):
    b, p = orig(n)
    C.memset(p, 0xAB, n)
    return b, p
_lib.new_bytes = filled
G = "tests/golden"
meta = json.load(open(os.path.join(G, "small.json"))); data = np.load(os.path.join(G, "small.npz"))
bad = 0
for rep in range(3):
    for i, m in enumerate(meta):
        a = data[f"in{i}"]; want = data[f"blob{i}"].tobytes()
        vr = tuple(m["value_range"]) if m["value_range"] else None
        b = P.mgard_compress(a, m["eb_rel"], m["dict_size"], value_range=vr)
        if b != want:
            bad += 1
            diff = [k for k in range(min(len(b), len(want))) if b[k] != want[k]]
            print("MISMATCH", rep, i, m["shape"], m["dict_size"], len(b), len(want), diff[:10], b[diff[0]:diff[0]+8].hex() if diff else "", flush=True)
print("bad", bad)
