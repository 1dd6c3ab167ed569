import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: larger configuration-scale cases")


@pytest.fixture(scope="session")
def small_cases():
    meta = json.load(open(os.path.join(GOLDEN, "small.json")))
    data = np.load(os.path.join(GOLDEN, "small.npz"))
    cases = []
    for i, m in enumerate(meta):
        c = dict(m)
        c["i"] = i
        c["input"] = data[f"in{i}"]
        c["coef"] = data[f"coef{i}"]
        c["recomp"] = data[f"recomp{i}"]
        c["blob"] = data[f"blob{i}"].tobytes()
        c["out"] = data[f"out{i}"]
        cases.append(c)
    return cases


@pytest.fixture(scope="session")
def huffman_golden():
    meta = json.load(open(os.path.join(GOLDEN, "huffman.json")))
    data = np.load(os.path.join(GOLDEN, "huffman.npz"))
    return meta, data


@pytest.fixture(scope="session")
def kat():
    return json.load(open(os.path.join(GOLDEN, "kat.json")))


@pytest.fixture(scope="session")
def corrupt_cases():
    return json.load(open(os.path.join(GOLDEN, "corrupt.json")))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def zfp_golden():
    """Fixed-rate coder vectors from the reference (tests/golden/gen_zfp_golden.py)."""
    meta = json.load(open(os.path.join(GOLDEN, "zfp.json")))
    data = np.load(os.path.join(GOLDEN, "zfp.npz"))
    cases = []
    for m in meta["cases"]:
        c = dict(m)
        i = m["id"]
        c["input"] = data[f"in{i}"]
        c["blob"] = data[f"blob{i}"].tobytes()
        c["out"] = data[f"out{i}"]
        cases.append(c)
    return cases, meta["errors"], data
