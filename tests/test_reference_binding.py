"""The INTEGRATION.md binding, exercised from the reference side.

integration/codec_binding.install() rebinds the UNMODIFIED reference's hpdr.mgard codec
(baseline/_ref, installed with pip --target) to libhpdr_b200.so; the reference's own public
calls (hpdr.mgard.mgard_compress / mgard_decompress with hpdr TensorData) must then reproduce
the blobs, reconstructions and exceptions the reference itself produced (tests/golden/).
"""
import hashlib
import importlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref_hpdr():
    if not os.path.isdir(os.path.join(REF, "hpdr")):
        pytest.skip("baseline/_ref (the reference install) is not present")
    sys.path.insert(0, REF)
    try:
        hpdr = importlib.import_module("hpdr")
        importlib.import_module("hpdr.mgard")
        yield hpdr
    finally:
        sys.path.remove(REF)


def test_binding_installs_on_the_reference(ref_hpdr):
    """The binding resolves every C-ABI symbol it calls and rebinds the reference's names
    (no GPU call: hpdr_ctx_create fails cleanly without a device)."""
    import ctypes as C

    from integration import codec_binding

    L = C.CDLL(codec_binding._LIB)
    for sym in ("hpdr_ctx_create", "hpdr_mgard_compress", "hpdr_mgard_fetch", "hpdr_mgard_peek",
                "hpdr_mgard_decompress", "hpdr_last_error"):
        assert hasattr(L, sym), sym
    codec = sys.modules["hpdr.mgard.codec"]
    assert callable(codec.mgard_compress) and callable(codec.mgard_decompress)


@pytest.mark.gpu
def test_reference_api_through_binding_matches_goldens(ref_hpdr, small_cases, corrupt_cases):
    from integration import codec_binding

    codec = sys.modules["hpdr.mgard.codec"]
    mg = sys.modules["hpdr.mgard"]
    prev = codec_binding.install(codec)
    try:
        TensorData, DType = codec.TensorData, codec.DType
        assert mg.mgard_compress is not prev[0]
        for c in small_cases:
            a = c["input"]
            u = TensorData(tuple(a.shape), DType.F32 if a.dtype == np.float32 else DType.F64, a)
            vr = tuple(c["value_range"]) if c["value_range"] else None
            blob = mg.mgard_compress(u, c["eb_rel"], c["dict_size"], value_range=vr)
            if blob != c["blob"]:   # say where (length, first differing byte, both tails)
                d = next((k for k in range(min(len(blob), len(c["blob"]))) if blob[k] != c["blob"][k]), None)
                again = mg.mgard_compress(u, c["eb_rel"], c["dict_size"], value_range=vr)
                pytest.fail(f"{c['shape']}: len {len(blob)} vs {len(c['blob'])}, first diff at {d}, "
                            f"tail {blob[-16:].hex()} vs {c['blob'][-16:].hex()}, repeat equal: {again == c['blob']}")
            y = mg.mgard_decompress(blob)
            assert isinstance(y, TensorData) and y.dtype == u.dtype and tuple(y.dims) == tuple(a.shape)
            assert np.array_equal(y.values.view(np.uint8), c["out"].view(np.uint8)), c["shape"]
        errors = sys.modules["hpdr.errors"]
        for name, c in corrupt_cases.items():
            blob = bytes.fromhex(c["hex"])
            if c["ok"]:
                out = mg.mgard_decompress(blob).values
                assert hashlib.sha256(out.tobytes()).hexdigest() == c["sha"], name
                continue
            exc = {"CorruptStreamError": errors.CorruptStreamError, "ValidationError": errors.ValidationError,
                   "OverflowError": OverflowError, "IndexError": IndexError, "ValueError": ValueError}[c["exc"]]
            with pytest.raises(exc) as ei:
                mg.mgard_decompress(blob)
            if c["exc"] == "CorruptStreamError":
                assert ei.value.bit_offset == c["bit_offset"], name
        # validation errors come out as the reference's class
        with pytest.raises(errors.ValidationError):
            mg.mgard_compress(TensorData((4,), DType.I32, np.zeros(4, np.int32)), 1e-3)
    finally:
        codec.mgard_compress, codec.mgard_decompress = prev
        mg.mgard_compress, mg.mgard_decompress = prev
