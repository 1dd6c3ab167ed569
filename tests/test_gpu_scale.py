"""Config-scale parity pins on the GPU (BASELINE configs at their full sizes).

Every field is rebuilt here from the seeded generators and checked against the pinned input
hash; blobs and reconstructions are checked against the sha256 of the reference's output
(tests/golden/configs.json: the reference itself; tests/golden/scale_pins.json: the C oracle,
which test_oracle_golden.py pins to the reference -- see gen_scale_pins.py):

* the north-star Target, 1024^3 fp32 rel 1e-4, through the pinned host path (M1) and through the
  streams pipeline (M2 container, 64 chunks, each chunk blob pinned);
* C3, NYX-like 6 fields x 4 bounds at 512^3;
* C4, first and last dim-0 slab of the 1024^3 fp64 field for 2, 4 and 8 GPUs (global range).
"""
import hashlib
import json
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import paper_2503_06322_b200 as P
from paper_2503_06322_b200 import synthetic as S

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _pins():
    pins = json.load(open(os.path.join(GOLDEN, "configs.json")))
    pins.update(json.load(open(os.path.join(GOLDEN, "scale_pins.json"))))
    return pins


def _sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def _pinned(a):
    import torch

    return torch.from_numpy(a).pin_memory()


def test_target_1024_m1_and_m2_match_pins():
    import torch

    from paper_2503_06322_b200 import pipeline as PL
    from paper_2503_06322_b200.container import read_container

    c = _pins()["T_smooth1024_f32_rel1e-4"]
    a = S.smooth_noise(tuple(c["shape"]), seed=0)
    assert S.sha256(a) == c["input_sha"], "input generator differs on this host"
    h_in = _pinned(a)
    h_blob = torch.empty(a.nbytes, dtype=torch.uint8).pin_memory()
    n = P.mgard_compress(h_in, c["eb_rel"], out=h_blob)
    assert n == c["blob_len"] and _sha(bytes(h_blob[:n].numpy())) == c["blob_sha"]
    h_out = torch.empty(a.shape, dtype=torch.float32).pin_memory()
    P.mgard_decompress(h_blob[:n], out=h_out)
    assert S.sha256(h_out.numpy()) == c["out_sha"]
    # M2: 16-plane chunks, each the reference blob of its chunk under the global range
    cont = PL.compress_pipelined(h_in, c["eb_rel"], chunk_planes=c["m2_chunk_planes"])
    h, payloads = read_container(cont)
    assert (h.vmin, h.vmax) == tuple(c["m2_value_range"])
    assert [_sha(bytes(p)) for p in payloads] == c["m2_chunk_sha"]
    y = PL.decompress_pipelined(cont)
    assert np.max(np.abs(y.astype(np.float64) - a)) <= c["eb_rel"] * (h.vmax - h.vmin)


def _nyx(field):
    return S.nyx_like((512,) * 3, field)


def test_c3_nyx_512_all_fields_and_bounds_match_pins():
    pins = _pins()
    with ProcessPoolExecutor(max_workers=min(6, os.cpu_count() or 1)) as ex:   # 6 x ~30 s of generation
        fields = dict(zip(S.NYX_FIELDS, ex.map(_nyx, S.NYX_FIELDS)))
    checked = 0
    for f, a in fields.items():
        for eb in (1e-2, 1e-3, 1e-4, 1e-5):
            c = pins[f"C3_{f}_512_{eb:g}"]
            assert S.sha256(a) == c["input_sha"], f
            blob = P.mgard_compress(a, eb)
            assert len(blob) == c["blob_len"] and _sha(blob) == c["blob_sha"], (f, eb)
            assert S.sha256(P.mgard_decompress(blob).values) == c["out_sha"], (f, eb)
            checked += 1
    assert checked == 24


@pytest.mark.parametrize("n", [2, 4, 8])
def test_c4_fp64_slabs_match_pins(n):
    pins = _pins()
    per = 1024 // n
    for k in sorted({0, n - 1}):
        c = pins[f"C4_smooth1024_f64_slab{k}of{n}"]
        a = S.smooth_noise((1024,) * 3, seed=0, dtype=np.float64, planes=(k * per, (k + 1) * per))
        assert S.sha256(a) == c["input_sha"]
        blob = P.mgard_compress(_pinned(a), c["eb_rel"], value_range=tuple(c["value_range"]))
        assert len(blob) == c["blob_len"] and _sha(blob) == c["blob_sha"], (k, n)
        assert S.sha256(P.mgard_decompress(blob).values) == c["out_sha"], (k, n)
        if n == 8 and k == 0:   # the one slab the reference itself produced (configs.json)
            ref = json.load(open(os.path.join(GOLDEN, "configs.json")))["C4_smooth1024_f64_slab0of8"]
            assert _sha(blob) == ref["blob_sha"]
