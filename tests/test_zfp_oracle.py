"""Pin the fixed-rate CPU oracle (oracle/zfp_oracle.c) against streams produced by the
reference hpdr/zfp.py itself (tests/golden/gen_zfp_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle.oracle import OracleError


def test_streams_bit_exact(zfp_golden, oracle):
    cases, _, _ = zfp_golden
    for c in cases:
        blob = oracle.zfp_compress(c["input"], c["rate"])
        assert len(blob) == c["len"]
        assert blob == c["blob"], (c["id"], c["dims"], c["dtype"], c["rate"], c["kind"])


def test_reconstruction_bit_exact(zfp_golden, oracle):
    cases, _, _ = zfp_golden
    for c in cases:
        out = oracle.zfp_decompress(c["blob"])
        assert out.dtype == c["out"].dtype and out.shape == c["out"].shape
        assert np.array_equal(out.view(np.uint8), c["out"].view(np.uint8)), c["id"]


def test_compressed_size_formula(zfp_golden, oracle):
    cases, _, _ = zfp_golden
    for c in cases:
        code = 0 if c["dtype"] == "f32" else 1
        assert oracle.zfp_compressed_size(c["dims"], code, c["rate"]) == c["len"]


def test_mutated_streams(zfp_golden, oracle):
    _, errors, data = zfp_golden
    codes = {None: 0, "CorruptStreamError": 2, "ValidationError": 1}
    for e in errors:
        if not e["case"].startswith("decode_"):
            continue
        name = e["case"][len("decode_"):]
        blob = data[f"mut_{name}"].tobytes()
        if e["raises"] is None:
            out = oracle.zfp_decompress(blob)
            assert np.array_equal(out.view(np.uint8), data[f"mutout_{name}"].view(np.uint8)), name
        else:
            with pytest.raises(OracleError) as ei:
                oracle.zfp_decompress(blob)
            assert ei.value.code == codes[e["raises"]], name
