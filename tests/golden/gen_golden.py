"""Generate golden vectors by running the REFERENCE itself (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_golden.py [--big]

Imports the reference package from /root/reference/pkg/src (read-only; it is
not available on the GPU box) and writes small fixtures next to this file:

* kat.json      -- SPEC / SURVEY §4 known-answer vectors, verified against the code
* small.npz     -- per-case inputs, reference blobs, coefficients, reconstructions
* huffman.npz   -- key streams and reference Huffman streams, codebook tables
* corrupt.json  -- mutated blobs and the exception class / bit_offset the reference raises
* configs.json  -- (--big) sha256 / length / CR / err of reference blobs at config scale
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from hpdr import huffman as H  # noqa: E402
from hpdr.errors import CorruptStreamError, ValidationError  # noqa: E402
from hpdr.exec_core import DType, TensorData, dem_exclusive_scan  # noqa: E402
from hpdr.mgard import build_hierarchy, decompose, mgard_compress, mgard_decompress, recompose  # noqa: E402
from hpdr.mgard.quantize import zigzag  # noqa: E402

from paper_2503_06322_b200 import synthetic as S  # noqa: E402


def td(a):
    return TensorData(a.shape, DType.F32 if a.dtype == np.float32 else DType.F64, a)


def kat():
    out = {}
    hs = {}
    for dims in ([5], [2], [9, 5], [1024], [129, 129, 129], [512, 512, 512], [128, 1024, 1024],
                 [4, 1024, 1024], [1, 17, 33], [5, 6, 7, 8]):
        h = build_hierarchy(dims)
        hs[str(dims)] = {"L": h.total_levels, "counts": [list(map(int, c)) for c in h.level_counts],
                         "owned": list(map(int, h.level_element_counts())),
                         "coarsest": list(map(int, h.coarsest_flat_indices()))[:64],
                         "maps_last": [list(map(int, h.index_maps[d][-1])) for d in range(len(dims))]}
    out["hierarchy"] = hs
    dec = {}
    for name, v in (("ramp", [0., 1, 2, 3, 4]), ("const", [3.] * 5), ("hat", [0., 0, 1, 0, 0])):
        a = np.array(v)
        h = build_hierarchy([5])
        c = decompose(td(a), h)
        dec[name] = {"in": v, "coef": c.values.tolist(), "rec": recompose(c, h).tolist()}
    out["decompose5"] = dec
    out["zigzag"] = zigzag(np.array([0, 1, -1, 2, -2])).tolist()
    cb = {}
    for name, f in (("5211", [5, 2, 1, 1]), ("single", [0, 7, 0]), ("two", [3, 3]), ("six", [1] * 6)):
        b = H.build_codebook(H.FrequencyTable(len(f), np.array(f)))
        cb[name] = {"freq": f, "lengths": b.lengths.tolist(), "codes": b.codes.tolist()}
    out["codebook"] = cb
    out["scan"] = dem_exclusive_scan(np.array([4, 7, 3])).tolist()
    out["histogram"] = H.histogram(np.array([1, 1, 2, 3], np.uint32), 4).counts.tolist()
    out["huffman_001"] = H.huffman_compress(np.array([0, 0, 1], np.uint32), 2).hex()
    try:
        H.build_codebook(H.FrequencyTable(40, np.array([1, 1] + [0] * 38)))
    except Exception as e:  # pragma: no cover
        out["codebook_err"] = type(e).__name__
    fib = [1, 1]
    while len(fib) < 40:
        fib.append(fib[-1] + fib[-2])
    try:
        H.build_codebook(H.FrequencyTable(40, np.array(fib)))
        out["fibonacci_err"] = None
    except ValidationError as e:
        out["fibonacci_err"] = str(e)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(out, f, indent=1)


SMALL_CASES = [
    # (shape, dtype, field, eb_rel, dict_size, value_range)
    ((5,), "f64", "rand", 1e-2, 4096, None),
    ((2,), "f32", "rand", 1e-2, 4096, None),
    ((3,), "f32", "rand", 1e-3, 4096, None),
    ((1000,), "f32", "rand", 1e-2, 4096, None),
    ((9, 5), "f64", "rand", 1e-3, 4096, None),
    ((65, 40), "f32", "smooth", 1e-4, 4096, None),
    ((12, 10, 9), "f64", "rand", 1e-3, 4096, None),
    ((16, 5, 7), "f64", "rand", 1e-4, 4096, None),
    ((4, 17, 8), "f32", "rand", 1e-3, 4096, None),
    ((9, 17, 1), "f32", "rand", 1e-2, 4096, None),
    ((1, 17, 33), "f32", "smooth", 1e-3, 4096, None),
    ((1, 1, 1), "f32", "rand", 1e-2, 4096, None),
    ((17, 17, 17), "f32", "grf", 1e-3, 4096, (0.0, 1.0)),
    ((33, 33, 33), "f32", "grf", 1e-3, 4096, None),
    ((33, 33, 33), "f32", "rand", 1e-3, 4096, None),
    ((32, 32, 32), "f32", "smooth", 1e-4, 4096, None),
    ((20, 24, 30), "f64", "smooth", 1e-5, 4096, None),
    ((16, 16, 16), "f32", "rand", 1e-5, 256, None),
    ((16, 16, 16), "f32", "grf", 1e-2, 65535, None),
    ((16, 16, 16), "f32", "grf", 1e-3, 2, None),
    ((5, 6, 7, 8), "f32", "rand", 1e-2, 4096, None),
    ((2, 2, 2, 2), "f32", "rand", 1e-2, 4096, None),
    ((6, 9, 10, 5), "f64", "rand", 1e-3, 4096, None),
    ((64, 33, 17), "f64", "smooth", 1e-4, 4096, None),
    ((40, 40, 40), "f32", "const", 1e-3, 4096, None),
    ((30, 31, 32), "f32", "ramp", 1e-3, 4096, None),
    ((24, 24, 24), "f32", "velocity", 1e-5, 4096, None),
    ((24, 24, 24), "f32", "density", 1e-2, 4096, None),
    ((24, 24, 24), "f64", "smooth", 1e-4, 4096, (-4.0, 12.0)),
]


def make_field(shape, dtype, field, seed):
    dt = np.float32 if dtype == "f32" else np.float64
    rng = np.random.default_rng(seed)
    if field == "rand":
        return rng.random(shape).astype(dt)
    if field == "smooth":
        return S.smooth_noise(shape, seed=seed, dtype=dt)
    if field == "grf":
        return S.grf(shape, m=4, seed=seed, dtype=dt)
    if field == "const":
        return np.full(shape, 3.25, dtype=dt)
    if field == "ramp":
        return (np.arange(int(np.prod(shape)), dtype=np.float64).reshape(shape) * 0.001).astype(dt)
    if field == "velocity":
        return S.nyx_like(shape, "velocity_x", seed=seed, dtype=dt)
    if field == "density":
        return S.nyx_like(shape, "baryon_density", seed=seed, dtype=dt)
    raise ValueError(field)


def small():
    arrays = {}
    meta = []
    for i, (shape, dtype, field, eb, dsz, vr) in enumerate(SMALL_CASES):
        a = make_field(shape, dtype, field, seed=100 + i)
        t = td(a)
        h = build_hierarchy(shape)
        c = decompose(t, h)
        blob = mgard_compress(t, eb, dict_size=dsz, value_range=vr)
        rec = mgard_decompress(blob).values
        arrays[f"in{i}"] = a
        arrays[f"coef{i}"] = c.values
        arrays[f"recomp{i}"] = recompose(c, h)
        arrays[f"blob{i}"] = np.frombuffer(blob, np.uint8)
        arrays[f"out{i}"] = rec
        meta.append({"shape": list(shape), "dtype": dtype, "field": field, "eb_rel": eb, "dict_size": dsz,
                     "value_range": vr, "blob_len": len(blob)})
    np.savez_compressed(os.path.join(HERE, "small.npz"), **arrays)
    with open(os.path.join(HERE, "small.json"), "w") as f:
        json.dump(meta, f, indent=1)


def huffman_fixtures():
    rng = np.random.default_rng(7)
    arrays = {}
    meta = []
    cases = [
        ("geometric", lambda: np.minimum(rng.geometric(0.3, 50000) - 1, 4095).astype(np.uint32), 4096),
        ("uniform", lambda: rng.integers(0, 256, 20000).astype(np.uint32), 256),
        ("zipf", lambda: np.minimum(rng.zipf(1.3, 30001) - 1, 1023).astype(np.uint32), 1024),
        ("single", lambda: np.full(5000, 17, np.uint32), 4096),
        ("empty", lambda: np.zeros(0, np.uint32), 4096),
        ("two", lambda: rng.integers(0, 2, 4097).astype(np.uint32), 2),
        ("one_sym", lambda: np.array([3], np.uint32), 8),
        ("deep", lambda: np.repeat(np.arange(22, dtype=np.uint32), [2 ** k for k in range(22)]), 64),
        ("wide", lambda: rng.integers(0, 65535, 70000).astype(np.uint32), 65535),
    ]
    for i, (name, gen, dsz) in enumerate(cases):
        k = gen()
        s = H.huffman_compress(k, dsz)
        back = H.huffman_decompress(s)
        assert np.array_equal(back, k)
        arrays[f"keys{i}"] = k
        arrays[f"stream{i}"] = np.frombuffer(s, np.uint8)
        meta.append({"name": name, "dict_size": dsz, "len": len(s)})
    cb = []
    for j in range(200):
        d = int(rng.integers(2, 300))
        cnt = rng.integers(0, 1000, d) * (rng.random(d) < 0.7)
        if np.count_nonzero(cnt) == 0:
            cnt[0] = 1
        b = H.build_codebook(H.FrequencyTable(d, cnt))
        arrays[f"cbcounts{j}"] = cnt.astype(np.int64)
        arrays[f"cblengths{j}"] = b.lengths
        arrays[f"cbcodes{j}"] = b.codes
        cb.append(d)
    np.savez_compressed(os.path.join(HERE, "huffman.npz"), **arrays)
    with open(os.path.join(HERE, "huffman.json"), "w") as f:
        json.dump({"streams": meta, "codebooks": cb}, f, indent=1)


def corrupt():
    a = S.grf((33, 33, 33), m=4, seed=5)
    blob = mgard_compress(td(a), 1e-3)
    rank = 3
    hdr = 1 + 8 * rank + 49
    # locate the Huffman stream and its packed payload
    n_out = int.from_bytes(blob[hdr:hdr + 8], "little")
    p = hdr + 8 + 16 * n_out
    n_co = int.from_bytes(blob[p:p + 8], "little")
    hpos = p + 8 + 8 * n_co
    dsz = int.from_bytes(blob[hpos:hpos + 2], "little")
    units_pos = hpos + 10 + dsz
    nunits = int.from_bytes(blob[units_pos:units_pos + 4], "little")
    packed_pos = units_pos + 4 + 8 * nunits + 8
    cases = {}

    def flip(b, pos, mask):
        bb = bytearray(b)
        bb[pos] ^= mask
        return bytes(bb)

    def setfield(b, pos, val, n):
        bb = bytearray(b)
        bb[pos:pos + n] = int(val).to_bytes(n, "little", signed=False)
        return bytes(bb)

    muts = {
        "ok": blob,
        "trailing7": blob + b"\x01" * 7,
        "trunc1": blob[:-1],
        "trunc20": blob[:-20],
        "trunc40": blob[:40],
        "trunc_in_outliers": blob[:hdr + 4],
        "trunc_in_lengths": blob[:hpos + 100],
        "trunc_in_offsets": blob[:units_pos + 20],
        "flip_bit": flip(blob, packed_pos + 1000, 0x10),
        "flip_byte": flip(blob, packed_pos + 5000, 0xFF),
        "flip_first": flip(blob, packed_pos, 0x80),
        "nsym_minus1": setfield(blob, hpos + 2, a.size - 1, 8),
        "levels99": setfield(blob, 1 + 8 * rank + 45, 99, 4),
        "dtype7": setfield(blob, 1 + 8 * rank, 7, 1),
        "units_short": setfield(blob, units_pos, max(0, nunits - 1), 4),
        "total_bits_big": setfield(blob, units_pos + 4 + 8 * nunits,
                                   8 * (len(blob) - packed_pos) + 9, 8),
        "total_bits_small": setfield(blob, units_pos + 4 + 8 * nunits, 50000, 8),
        "lengths_zero": blob[:hpos + 10] + bytes(dsz) + blob[hpos + 10 + dsz:],
        "dict_small": setfield(blob, 1 + 8 * rank + 9, 3, 4),
        "mgard_dict_big": setfield(blob, 1 + 8 * rank + 9, 60000, 4),
        "offset_skew": setfield(blob, units_pos + 4 + 8 * 3, 12345, 8),
        "length_40": blob[:hpos + 10 + 5] + bytes([40]) + blob[hpos + 10 + 6:],
        "empty": b"",
        "only_rank": bytes([3]),
    }
    for name, m in muts.items():
        rec = {"hex": m.hex()}
        try:
            out = mgard_decompress(m).values
            rec.update(ok=True, sha=hashlib.sha256(out.tobytes()).hexdigest())
        except CorruptStreamError as e:
            rec.update(ok=False, exc="CorruptStreamError", bit_offset=e.bit_offset)
        except ValidationError:
            rec.update(ok=False, exc="ValidationError")
        except Exception as e:
            rec.update(ok=False, exc=type(e).__name__)
        cases[name] = rec
    with open(os.path.join(HERE, "corrupt.json"), "w") as f:
        json.dump(cases, f)


def config_case(name, a, eb, value_range=None):
    t0 = time.time()
    blob = mgard_compress(td(a), eb, value_range=value_range)
    t1 = time.time()
    rec = mgard_decompress(blob).values
    t2 = time.time()
    rng_ = (value_range[1] - value_range[0]) if value_range else float(a.max()) - float(a.min())
    err = float(np.max(np.abs(rec.astype(np.float64) - a.astype(np.float64))))
    r = {"name": name, "shape": list(a.shape), "dtype": str(a.dtype), "eb_rel": eb,
         "value_range": value_range, "input_sha": S.sha256(a), "blob_sha": hashlib.sha256(blob).hexdigest(),
         "blob_len": len(blob), "out_sha": S.sha256(rec), "cr": a.nbytes / len(blob),
         "err_over_eb": err / (eb * rng_) if rng_ > 0 else 0.0,
         "ref_compress_s": t1 - t0, "ref_decompress_s": t2 - t1}
    print(json.dumps(r), flush=True)
    return r


def big():
    path = os.path.join(HERE, "configs.json")
    done = json.load(open(path)) if os.path.exists(path) else {}
    todo = [
        ("C1_grf129_abs1e-3", lambda: (S.grf((129,) * 3, m=8, seed=0), 1e-3, (0.0, 1.0))),
        ("C2_smooth513_rel1e-4", lambda: (S.smooth_noise((513,) * 3, seed=0), 1e-4, None)),
    ]
    for f in S.NYX_FIELDS:
        for eb in (1e-2, 1e-3, 1e-4, 1e-5):
            todo.append((f"C3_{f}_129_{eb:g}", lambda f=f, eb=eb: (S.nyx_like((129,) * 3, f), eb, None)))
    todo.append(("C3_temperature_512_1e-3", lambda: (S.nyx_like((512,) * 3, "temperature"), 1e-3, None)))
    todo.append(("C4_smooth1024_f64_slab0of8", lambda: (
        S.smooth_noise((1024, 1024, 1024), seed=0, dtype=np.float64)[:128].copy(), 1e-4, "global")))
    for name, gen in todo:
        if name in done:
            continue
        a, eb, vr = gen()
        if vr == "global":
            vr = C4_RANGE
        done[name] = config_case(name, a, eb, vr)
        with open(path, "w") as f:
            json.dump(done, f, indent=1)


# global range of the 1024^3 fp64 C4 field: computed once by gen (min/max over all slabs)
C4_RANGE = None


def c4_range():
    global C4_RANGE
    a = S.smooth_noise((1024, 1024, 1024), seed=0, dtype=np.float64)
    C4_RANGE = (float(a.min()), float(a.max()))
    del a


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    kat()
    small()
    huffman_fixtures()
    corrupt()
    if args.big:
        c4_range()
        big()
