"""Config-scale parity pins (sha256 of blobs and reconstructions) -> tests/golden/scale_pins.json.

The pins come from the C oracle (oracle/mgard_oracle.c), which is itself pinned to the
reference: tests/test_oracle_golden.py checks it against blobs the reference produced
(gen_golden.py, including C2 513^3, C3 temperature 512^3 and the C4 1/8 slab), so a pin here
is the reference's output for these inputs.  Running the reference itself at 1024^3 needs
~75 GB of RSS and ~10 min per direction on one core (SURVEY App. C probe 18), more than this
container has.

Inputs are rebuilt on the GPU box from the seeded, SIMD-invariant generators
(paper_2503_06322_b200/synthetic.py); every pin carries the input's sha256 so a generator
difference shows up as such.

    python tests/golden/gen_scale_pins.py [--only NAME_PREFIX] [--threads 8]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2503_06322_b200 import synthetic as S  # noqa: E402

PATH = os.path.join(HERE, "scale_pins.json")
T_SHAPE = (1024, 1024, 1024)
T_EB = 1e-4
T_CHUNK_PLANES = 16          # the M2 container pin: 64 chunks of 16 planes (64 MB of fp32)
C4_SHAPE = (1024, 1024, 1024)
C4_EB = 1e-4


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def case(a, eb, value_range=None):
    t0 = time.time()
    blob = O.mgard_compress(a, eb, value_range=value_range)
    t1 = time.time()
    rec = O.mgard_decompress(blob)
    t2 = time.time()
    rng_ = (value_range[1] - value_range[0]) if value_range else float(a.max()) - float(a.min())
    err = float(np.max(np.abs(rec.astype(np.float64) - a.astype(np.float64))))
    return {"shape": list(a.shape), "dtype": str(a.dtype), "eb_rel": eb,
            "value_range": list(value_range) if value_range else None, "input_sha": S.sha256(a),
            "blob_sha": sha(blob), "blob_len": len(blob), "out_sha": S.sha256(rec), "cr": a.nbytes / len(blob),
            "err_over_eb": err / (eb * rng_) if rng_ > 0 else 0.0,
            "oracle_compress_s": t1 - t0, "oracle_decompress_s": t2 - t1}


def c4_range():
    cfg = json.load(open(os.path.join(HERE, "configs.json")))["C4_smooth1024_f64_slab0of8"]
    return tuple(cfg["value_range"])


def jobs():
    # the north-star Target: 1024^3 fp32, relative L-inf 1e-4 (M1: one blob) ...
    def target():
        a = S.smooth_noise(T_SHAPE, seed=0)
        r = case(a, T_EB)
        # ... and the M2 container: every 16-plane chunk a blob with the global range
        vr = (float(a.min()), float(a.max()))
        r["m2_chunk_planes"] = T_CHUNK_PLANES
        r["m2_value_range"] = list(vr)
        r["m2_chunk_sha"] = [sha(O.mgard_compress(a[p:p + T_CHUNK_PLANES], T_EB, value_range=vr))
                             for p in range(0, T_SHAPE[0], T_CHUNK_PLANES)]
        return r

    yield "T_smooth1024_f32_rel1e-4", target
    # C3: NYX-like 6 fields x 4 bounds at 512^3
    for f in S.NYX_FIELDS:
        for eb in (1e-2, 1e-3, 1e-4, 1e-5):
            yield f"C3_{f}_512_{eb:g}", (lambda f=f, eb=eb: case(S.nyx_like((512,) * 3, f), eb))
    # C4: first and last dim-0 slab of the 1024^3 fp64 field for 2, 4, 8 GPUs, global range
    for n in (2, 4, 8):
        per = C4_SHAPE[0] // n
        for k in sorted({0, n - 1}):
            yield (f"C4_smooth1024_f64_slab{k}of{n}",
                   lambda per=per, k=k: case(S.smooth_noise(C4_SHAPE, seed=0, dtype=np.float64,
                                                            planes=(k * per, (k + 1) * per)), C4_EB, c4_range()))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    O.set_threads(args.threads)
    done = json.load(open(PATH)) if os.path.exists(PATH) else {}
    for name, fn in jobs():
        if name in done or not name.startswith(args.only):
            continue
        t = time.time()
        done[name] = {"name": name, **fn()}
        print(name, f"{time.time() - t:.1f}s", done[name]["blob_len"], done[name]["err_over_eb"], flush=True)
        with open(PATH, "w") as f:
            json.dump(done, f, indent=1)


if __name__ == "__main__":
    main()
