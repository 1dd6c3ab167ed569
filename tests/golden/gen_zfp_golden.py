"""Generate fixed-rate (zfp.py) golden vectors by running the REFERENCE itself (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/gen_zfp_golden.py

Imports /root/reference/pkg/src/hpdr/zfp.py (read-only, absent on the GPU box) and writes

* zfp.npz   -- inputs, reference streams and reference reconstructions per case
* zfp.json  -- case list (dims, dtype, rate, kind), stream sizes, and the exception class the
               reference raises on invalid inputs / mutated streams
"""
from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from hpdr import zfp as Z  # noqa: E402
from hpdr.exec_core import DType, TensorData  # noqa: E402


def td(a):
    return TensorData(a.shape, DType.F32 if a.dtype == np.float32 else DType.F64, a)


def field(rng, dims, dt, kind):
    """Input families: uniform, large magnitude, mixed tiny/subnormal with zeros, all-zero,
    smooth ramp, negative constant, powers of two (exponent guard edges)."""
    a = rng.random(dims) * 2 - 1
    if kind == "big":
        a = a * (1e300 if dt == np.float64 else 3e38)
    elif kind == "tiny":
        tiny = 1e-310 if dt == np.float64 else 1e-41
        a = a * np.where(rng.random(dims) < 0.5, tiny, 1.0)
        a.reshape(-1)[::5] = 0.0
    elif kind == "zero":
        a = np.zeros(dims)
    elif kind == "ramp":
        a = np.arange(int(np.prod(dims)), dtype=np.float64).reshape(dims) / 7.0 - 3.0
    elif kind == "const":
        a = np.full(dims, -2.5)
    elif kind == "pow2":
        a = np.ldexp(1.0, rng.integers(-20, 20, size=dims)) * np.where(rng.random(dims) < 0.5, -1, 1)
    return np.ascontiguousarray(a.astype(dt))


def main():
    rng = np.random.default_rng(2503)
    arrays, cases = {}, []
    shapes = [(1,), (4,), (5,), (17,), (64,), (4, 4), (5, 7), (9, 13), (1, 33), (4, 4, 4), (5, 6, 7),
              (13, 9, 17), (1, 1, 9), (33, 17, 20)]
    kinds = ["uniform", "big", "tiny", "zero", "ramp", "const", "pow2"]
    i = 0
    for dims in shapes:
        for dt in (np.float32, np.float64):
            q = 32 if dt == np.float32 else 64
            for rate in (1, 5, 16, q):
                for kind in kinds:
                    if kind in ("zero", "const") and rate not in (5, q):
                        continue
                    a = field(rng, dims, dt, kind)
                    blob = Z.zfp_compress(td(a), rate)
                    back = Z.zfp_decompress(blob).values
                    assert len(blob) == Z.compressed_size(dims, td(a).dtype, rate)
                    arrays[f"in{i}"] = a
                    arrays[f"blob{i}"] = np.frombuffer(blob, np.uint8)
                    arrays[f"out{i}"] = back
                    cases.append({"id": i, "dims": list(dims), "dtype": "f32" if dt == np.float32 else "f64",
                                  "rate": rate, "kind": kind, "len": len(blob)})
                    i += 1

    # invalid inputs (zfp.py:61-62 rate range, :94-95 rank, :134-135 non-finite, :285-286 dtype)
    errors = []

    def expect(name, fn):
        try:
            fn()
            errors.append({"case": name, "raises": None})
        except Exception as e:  # noqa: BLE001
            errors.append({"case": name, "raises": type(e).__name__})

    f = np.ones((4, 4), np.float32)
    expect("rate0", lambda: Z.zfp_compress(td(f), 0))
    expect("rate33_f32", lambda: Z.zfp_compress(td(f), 33))
    expect("rate64_f64", lambda: Z.zfp_compress(td(f.astype(np.float64)), 64))
    expect("rate65_f64", lambda: Z.zfp_compress(td(f.astype(np.float64)), 65))
    expect("rank4", lambda: Z.zfp_compress(td(np.ones((2, 2, 2, 2), np.float32)), 8))
    nanf = f.copy()
    nanf[1, 2] = np.nan
    expect("nan", lambda: Z.zfp_compress(td(nanf), 8))
    inff = f.copy()
    inff[3, 3] = -np.inf
    expect("inf", lambda: Z.zfp_compress(td(inff), 8))
    expect("int_dtype", lambda: Z.zfp_compress(TensorData((4,), DType.I32, np.ones(4, np.int32)), 8))

    good = Z.zfp_compress(td(np.linspace(-1, 1, 5 * 6 * 7, dtype=np.float32).reshape(5, 6, 7)), 9)
    arrays["mut_base"] = np.frombuffer(good, np.uint8)
    muts = {
        "empty": b"",
        "short_header": good[:2],
        "rank0": bytes([0]) + good[1:],
        "rank4": bytes([4]) + good[1:],
        "dtype7": good[:1] + bytes([7]) + good[2:],
        "dtype_int": good[:1] + bytes([4]) + good[2:],
        "rate0": good[:2] + bytes([0]) + good[3:],
        "rate33": good[:2] + bytes([33]) + good[3:],
        "truncated_payload": good[:-1],
        "trailing_bytes": good + b"\x00\x01\x02",
        "flipped_bits": bytes(b ^ 0x5A if 40 <= k < 60 else b for k, b in enumerate(good)),
    }
    for name, data in muts.items():
        arrays[f"mut_{name}"] = np.frombuffer(data, np.uint8)
        try:
            out = Z.zfp_decompress(data).values
            arrays[f"mutout_{name}"] = out
            errors.append({"case": "decode_" + name, "raises": None})
        except Exception as e:  # noqa: BLE001
            errors.append({"case": "decode_" + name, "raises": type(e).__name__})

    np.savez_compressed(os.path.join(HERE, "zfp.npz"), **arrays)
    with open(os.path.join(HERE, "zfp.json"), "w") as fh:
        json.dump({"source": "hpdr/zfp.py (reference, run in the build container)", "cases": cases,
                   "errors": errors}, fh, indent=1)
    print(f"{len(cases)} cases, {len(errors)} error probes")


if __name__ == "__main__":
    main()
