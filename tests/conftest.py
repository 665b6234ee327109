import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    # same seed convention as the reference suite (pkg/tests/conftest.py:8-10)
    return np.random.default_rng(0xC0FFEE)


def load_golden_streams():
    z = np.load(os.path.join(GOLDEN, "streams.npz"))
    meta = json.loads(str(z["meta"]))
    inputs, streams = z["inputs"], z["streams"]
    io = so = 0
    out = []
    for m in meta:
        data = inputs[io: io + m["input_len"]].tobytes()
        stream = streams[so: so + m["stream_len"]].tobytes()
        io += m["input_len"]
        so += m["stream_len"]
        out.append((m, data, stream))
    return out


def load_golden_codebooks():
    z = np.load(os.path.join(GOLDEN, "codebooks.npz"))
    return z["hists"], z["lengths"]


def load_golden_corruptions():
    with open(os.path.join(GOLDEN, "corruptions.json")) as f:
        return json.load(f)


def reference_lmc():
    """The live reference package (build container only) or None."""
    if not os.path.isdir(REFERENCE_SRC):
        return None
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    try:
        import lmc  # noqa: F401
        return lmc
    except Exception:
        return None
