import ctypes as C, importlib, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
REF = os.path.join(os.getcwd(), "baseline", "_ref"); sys.path.insert(0, REF)
hpdr = importlib.import_module("hpdr"); importlib.import_module("hpdr.mgard")
from integration import codec_binding
codec = sys.modules["hpdr.mgard.codec"]; mg = sys.modules["hpdr.mgard"]
G = "tests/golden"
meta = json.load(open(os.path.join(G, "small.json"))); data = np.load(os.path.join(G, "small.npz"))
codec_binding.install(codec)
bad = 0
for i, m in enumerate(meta[:8]):
    a = data[f"in{i}"]; want = data[f"blob{i}"].tobytes()
    u = codec.TensorData(tuple(a.shape), codec.DType.F32 if a.dtype == np.float32 else codec.DType.F64, a)
    vr = tuple(m["value_range"]) if m["value_range"] else None
    b = mg.mgard_compress(u, m["eb_rel"], m["dict_size"], value_range=vr)
    bad += b != want
    y = mg.mgard_decompress(b)
print("bad", bad)
