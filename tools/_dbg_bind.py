import ctypes as C, importlib, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
REF = os.path.join(os.getcwd(), "baseline", "_ref"); sys.path.insert(0, REF)
hpdr = importlib.import_module("hpdr"); importlib.import_module("hpdr.mgard")
from integration import codec_binding
codec = sys.modules["hpdr.mgard.codec"]; mg = sys.modules["hpdr.mgard"]
G = "tests/golden"
meta = json.load(open(os.path.join(G, "small.json"))); data = np.load(os.path.join(G, "small.npz"))
for trial in range(4):
    # dirty the device allocator: fill and free big buffers
    x = torch.full((1 << 28,), 0x5A5A5A5A, dtype=torch.int32, device="cuda"); torch.cuda.synchronize(); del x
    torch.cuda.empty_cache()
    prev = codec_binding.install(codec)
    bad = 0
    for i, m in enumerate(meta):
        a = data[f"in{i}"]; want = data[f"blob{i}"].tobytes()
        u = codec.TensorData(tuple(a.shape), codec.DType.F32 if a.dtype == np.float32 else codec.DType.F64, a)
        vr = tuple(m["value_range"]) if m["value_range"] else None
        b = mg.mgard_compress(u, m["eb_rel"], m["dict_size"], value_range=vr)
        if b != want:
            bad += 1
            diff = [k for k in range(min(len(b), len(want))) if b[k] != want[k]]
            print("MISMATCH", trial, i, m["shape"], m["dict_size"], m["value_range"], len(b), len(want), diff[:12],
                  b[diff[0]:diff[0] + 8].hex() if diff else "", want[diff[0]:diff[0] + 8].hex() if diff else "", flush=True)
    print("trial", trial, "bad", bad, flush=True)
