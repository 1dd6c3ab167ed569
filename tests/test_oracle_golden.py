"""Pin the CPU oracle (oracle/mgard_oracle.c) against vectors produced by the reference
itself (tests/golden/gen_golden.py).  CPU only."""
import hashlib

import numpy as np
import pytest


def test_small_blobs_bit_exact(small_cases, oracle):
    for c in small_cases:
        vr = tuple(c["value_range"]) if c["value_range"] else None
        blob = oracle.mgard_compress(c["input"], c["eb_rel"], c["dict_size"], value_range=vr)
        assert blob == c["blob"], (c["i"], c["shape"], len(blob), len(c["blob"]))


def test_small_coefficients_bit_exact(small_cases, oracle):
    for c in small_cases:
        coef, _, _ = oracle.decompose(c["input"])
        assert np.array_equal(coef.view(np.uint64), c["coef"].view(np.uint64)), c["i"]
        rec = oracle.recompose(c["coef"])
        assert np.array_equal(rec.view(np.uint64), c["recomp"].view(np.uint64)), c["i"]


def test_small_decompress_bit_exact(small_cases, oracle):
    for c in small_cases:
        out = oracle.mgard_decompress(c["blob"])
        assert out.dtype == c["out"].dtype
        assert np.array_equal(out.view(np.uint8), c["out"].view(np.uint8)), c["i"]


def test_huffman_streams(huffman_golden, oracle):
    meta, data = huffman_golden
    for i, m in enumerate(meta["streams"]):
        keys = data[f"keys{i}"]
        s = oracle.huffman_compress(keys, m["dict_size"])
        assert s == data[f"stream{i}"].tobytes(), m["name"]
        back = oracle.huffman_decompress(s)
        assert np.array_equal(back, keys)


def test_codebooks(huffman_golden, oracle):
    meta, data = huffman_golden
    for j, d in enumerate(meta["codebooks"]):
        lens, codes = oracle.build_codebook(data[f"cbcounts{j}"], d)
        assert np.array_equal(lens, data[f"cblengths{j}"]), j
        assert np.array_equal(codes, data[f"cbcodes{j}"]), j


def test_kat_vectors(kat, oracle):
    for name, v in kat["decompose5"].items():
        coef, _, _ = oracle.decompose(np.array(v["in"], np.float64))
        assert coef.tolist() == v["coef"], name
        assert oracle.recompose(coef).tolist() == v["rec"], name
    for name, v in kat["codebook"].items():
        lens, codes = oracle.build_codebook(np.array(v["freq"]), len(v["freq"]))
        assert lens.tolist() == v["lengths"] and codes.tolist() == v["codes"], name
    assert oracle.huffman_compress(np.array([0, 0, 1], np.uint32), 2).hex() == kat["huffman_001"]
    for dims, h in kat["hierarchy"].items():
        dims = eval(dims)
        L, counts = oracle.hierarchy(dims)
        assert L == h["L"] and counts.tolist() == h["counts"], dims
        idx = oracle.coarsest_indices(dims)
        assert idx.tolist()[:64] == h["coarsest"], dims


def test_corrupt_streams(corrupt_cases, oracle):
    """The oracle reproduces the reference's accept / reject decisions and bit offsets."""
    for name, c in corrupt_cases.items():
        blob = bytes.fromhex(c["hex"])
        if c["ok"]:
            out = oracle.mgard_decompress(blob)
            assert hashlib.sha256(out.tobytes()).hexdigest() == c["sha"], name
        elif c["exc"] == "CorruptStreamError" and name not in ("empty",):
            with pytest.raises(oracle.OracleError) as ei:
                oracle.mgard_decompress(blob)
            assert ei.value.code == oracle.CORRUPT, name
            if c["bit_offset"] >= 0:
                assert ei.value.bit_offset == c["bit_offset"], name


def test_thread_count_invariance(small_cases, oracle):
    c = small_cases[13]
    oracle.set_threads(1)
    a = oracle.mgard_compress(c["input"], c["eb_rel"])
    oracle.set_threads(4)
    b = oracle.mgard_compress(c["input"], c["eb_rel"])
    oracle.set_threads(1)
    assert a == b == c["blob"]
