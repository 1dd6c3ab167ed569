"""Fixed-rate block coder (hpdr/zfp.py) on the GPU: byte parity with streams the reference produced
(tests/golden/zfp.npz), with the C oracle at configuration scale, and the reference's error classes.
Needs a B200: run with -m gpu."""
import numpy as np
import pytest

from paper_2503_06322_b200 import synthetic as S
from paper_2503_06322_b200 import zfp as Z
from paper_2503_06322_b200.errors import CorruptStreamError, ValidationError
from paper_2503_06322_b200.tensor import DType, TensorData

pytestmark = pytest.mark.gpu

ERR = {"ValidationError": ValidationError, "CorruptStreamError": CorruptStreamError}


def test_streams_match_reference(zfp_golden):
    cases, _, _ = zfp_golden
    for c in cases:
        blob = Z.zfp_compress(c["input"], c["rate"])
        assert len(blob) == c["len"] == Z.compressed_size(c["dims"], DType(c["dtype"]), c["rate"])
        assert blob == c["blob"], (c["id"], c["dims"], c["dtype"], c["rate"], c["kind"])


def test_reconstruction_matches_reference(zfp_golden):
    cases, _, _ = zfp_golden
    for c in cases:
        out = Z.zfp_decompress(c["blob"]).values
        assert out.dtype == c["out"].dtype and out.shape == c["out"].shape
        assert np.array_equal(out.view(np.uint8), c["out"].view(np.uint8)), (c["id"], c["kind"])


def test_tensor_data_and_device_buffers(zfp_golden):
    torch = pytest.importorskip("torch")
    cases, _, _ = zfp_golden
    for c in cases[::17]:
        a = c["input"]
        td = TensorData(a.shape, DType(c["dtype"]), a)
        assert Z.zfp_compress(td, c["rate"]) == c["blob"]
        dev_in = torch.from_numpy(a.copy()).cuda()
        dev_out = torch.empty(c["len"], dtype=torch.uint8, device="cuda")
        assert Z.zfp_compress(dev_in, c["rate"], out=dev_out) == c["len"]
        assert bytes(dev_out.cpu().numpy()) == c["blob"]
        dec = torch.empty(a.shape, dtype=dev_in.dtype, device="cuda")
        Z.zfp_decompress(dev_out, out=dec)
        assert np.array_equal(dec.cpu().numpy().view(np.uint8), c["out"].view(np.uint8))


def test_invalid_inputs_raise_like_reference(zfp_golden):
    _, errors, _ = zfp_golden
    want = {e["case"]: e["raises"] for e in errors}
    f = np.ones((4, 4), np.float32)
    nan = f.copy()
    nan[1, 2] = np.nan
    inf = f.copy()
    inf[3, 3] = -np.inf
    probes = {
        "rate0": lambda: Z.zfp_compress(f, 0),
        "rate33_f32": lambda: Z.zfp_compress(f, 33),
        "rate64_f64": lambda: Z.zfp_compress(f.astype(np.float64), 64),
        "rate65_f64": lambda: Z.zfp_compress(f.astype(np.float64), 65),
        "rank4": lambda: Z.zfp_compress(np.ones((2, 2, 2, 2), np.float32), 8),
        "nan": lambda: Z.zfp_compress(nan, 8),
        "inf": lambda: Z.zfp_compress(inf, 8),
        "int_dtype": lambda: Z.zfp_compress(np.ones(4, np.int32), 8),
    }
    for name, fn in probes.items():
        if want[name] is None:
            fn()
        else:
            with pytest.raises(ERR[want[name]]):
                fn()


def test_mutated_streams_like_reference(zfp_golden):
    _, errors, data = zfp_golden
    for e in errors:
        if not e["case"].startswith("decode_"):
            continue
        name = e["case"][len("decode_"):]
        blob = data[f"mut_{name}"].tobytes()
        if e["raises"] is None:
            out = Z.zfp_decompress(blob).values
            assert np.array_equal(out.view(np.uint8), data[f"mutout_{name}"].view(np.uint8)), name
        else:
            with pytest.raises(ERR[e["raises"]]):
                Z.zfp_decompress(blob)


@pytest.mark.parametrize("dims,dtype,rate", [((513, 513, 513), np.float32, 16), ((257, 129, 131), np.float64, 40),
                                             ((1031, 1029), np.float32, 7), (((1 << 20) + 3,), np.float64, 12)])
def test_config_scale_matches_oracle(oracle, dims, dtype, rate):
    """Whole streams at configuration scale (C2 = 513^3 fp32) byte-compared with the C oracle;
    the host path here is the streamed one (dim-0 slabs, overlapped copies)."""
    oracle.set_threads(16)
    a = S.smooth_noise(dims, seed=3, dtype=dtype) if len(dims) == 3 else \
        (np.random.default_rng(1).random(dims) * 2 - 1).astype(dtype)
    blob = Z.zfp_compress(a, rate)
    ref = oracle.zfp_compress(a, rate)
    assert len(blob) == len(ref)
    assert blob == ref
    back = Z.zfp_decompress(blob).values
    assert np.array_equal(back.view(np.uint8), oracle.zfp_decompress(ref).view(np.uint8))


def test_wide_offset_variant_matches_reference(zfp_golden):
    """The int64-offset kernels (blocks spanning > 2^31 elements) on the golden cases, forced."""
    import subprocess
    import sys

    code = (
        "import numpy as np, sys; sys.path.insert(0, '.');"
        "from paper_2503_06322_b200 import zfp as Z;"
        "d = np.load('tests/golden/zfp.npz'); import json;"
        "m = json.load(open('tests/golden/zfp.json'))['cases'];"
        "bad = [c['id'] for c in m[::5] if Z.zfp_compress(d['in%d' % c['id']], c['rate']) != d['blob%d' % c['id']].tobytes()"
        " or not np.array_equal(Z.zfp_decompress(d['blob%d' % c['id']].tobytes()).values.view(np.uint8),"
        " d['out%d' % c['id']].view(np.uint8))];"
        "print('BAD', bad)"
    )
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, HPDR_ZFP_WIDE="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "BAD []" in r.stdout, r.stdout


def _slabs(a, planes):
    out, p = [], 0
    for n in planes:
        out.append(np.ascontiguousarray(a[p:p + n]))
        p += n
    return out


@pytest.mark.parametrize("dims,dtype,rate,chunks", [((257, 129, 131), np.float32, 16, None),
                                                    ((130, 66, 35), np.float64, 40, [7, 64, 1, 58]),
                                                    ((1031, 1029), np.float32, 9, [500, 531])])
def test_pipeline_container_matches_per_slab_streams(oracle, dims, dtype, rate, chunks):
    """The fixed-rate reducer through the streams pipeline: an HPDR container (pipeline id 1) whose
    chunk payloads are byte-identical to the reference stream of each slab."""
    import torch

    from paper_2503_06322_b200 import pipeline as PL
    from paper_2503_06322_b200.container import PIPELINE_ZFP, read_container

    oracle.set_threads(16)
    a = (np.random.default_rng(7).random(dims) * 2 - 1).astype(dtype)
    pin = torch.from_numpy(a).pin_memory()
    data, tr = Z.compress_pipelined(pin, rate, chunks=chunks, trace=True, chunk_planes=0 if chunks else 40)
    h, pays = read_container(data)
    assert h.pipeline == PIPELINE_ZFP and h.rate == rate and h.dims == dims
    planes = [c.raw_size // int(np.prod(dims[1:])) for c in h.chunks]
    if chunks:
        assert planes == chunks
    assert tr.shape == (len(planes), 6) and np.all(tr[:, 3] >= tr[:, 2])
    for slab, p in zip(_slabs(a, planes), pays):
        assert bytes(p) == oracle.zfp_compress(slab, rate)
    back = PL.decompress_pipelined(data)
    ref = np.concatenate([oracle.zfp_decompress(bytes(p)) for p in pays])
    assert np.array_equal(np.asarray(back.values if hasattr(back, "values") else back).view(np.uint8),
                          ref.view(np.uint8))
    # device-resident input and output
    dev = torch.from_numpy(a).cuda()
    assert Z.compress_pipelined(dev, rate, chunks=chunks, chunk_planes=0 if chunks else 40) == data
    dout = torch.empty(dims, dtype=dev.dtype, device="cuda")
    PL.decompress_pipelined(data, out=dout)
    assert np.array_equal(dout.cpu().numpy().view(np.uint8), ref.view(np.uint8))


def test_pipeline_container_errors():
    """Fixed-rate container: a non-finite chunk raises ValidationError; a corrupted header (CRC) or a
    truncated container raise FormatError; a chunk stream that fails its own checks raises the
    reducer's error."""
    from paper_2503_06322_b200 import pipeline as PL
    from paper_2503_06322_b200.errors import FormatError

    a = (np.random.default_rng(3).random((40, 33, 17)) * 2 - 1).astype(np.float32)
    bad = a.copy()
    bad[37, 5, 5] = np.inf
    with pytest.raises(ValidationError):
        Z.compress_pipelined(bad, 12, chunk_planes=8)
    data = Z.compress_pipelined(a, 12, chunk_planes=8)
    hdr = bytearray(data)
    hdr[10] ^= 0x40   # inside the dims: CRC mismatch
    with pytest.raises(FormatError):
        PL.decompress_pipelined(bytes(hdr))
    with pytest.raises(FormatError):
        PL.decompress_pipelined(data[: len(data) - 5])
    from paper_2503_06322_b200.container import read_container

    h, pays = read_container(data)
    # a chunk stream whose own header disagrees with the container (rate byte of chunk 0)
    off = len(data) - sum(c.payload_size for c in h.chunks) + h.chunks[0].payload_offset
    mut = bytearray(data)
    mut[off + 2] = 13   # the chunk's own checks (zfp.py:333-334) or the container's consistency check
    with pytest.raises((FormatError, CorruptStreamError)):
        PL.decompress_pipelined(bytes(mut))
