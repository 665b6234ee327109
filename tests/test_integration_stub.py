"""The ctypes binding INTEGRATION.md proposes for the reference works as written.

The stub is extracted from INTEGRATION.md, its package-relative imports are
pointed at this repo's mirrors of ``lmc.errors`` / ``lmc.types`` (same class
names), and it is executed against the in-tree liblmc_b200.so.
"""
import os
import re
import types

import numpy as np
import pytest

from conftest import ROOT, load_golden_streams

LIB = os.path.join(ROOT, "paper_2505_09810_b200", "liblmc_b200.so")


def _load_stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "_b200.py" in b)
    code = code.replace("from .errors import", "from paper_2505_09810_b200.errors import")
    code = code.replace("from .types import", "from paper_2505_09810_b200.types import")
    os.environ["LMC_B200_LIB"] = LIB
    mod = types.ModuleType("lmc_b200_stub")
    exec(compile(code, "INTEGRATION.md:_b200.py", "exec"), mod.__dict__)
    return mod


def test_stub_binds_library():
    m = _load_stub()
    for name in ("lmcg_compress_host", "lmcg_decompress_host", "lmcg_create", "lmcg_last_error"):
        assert hasattr(m._lib, name)


@pytest.mark.gpu
def test_stub_round_trip_and_errors():
    from oracle import oracle as O
    from paper_2505_09810_b200.errors import CorruptStreamError, UnsupportedFormatError
    from paper_2505_09810_b200.types import ElementType, TensorBuffer

    m = _load_stub()
    rng = np.random.default_rng(5)
    raw = (rng.normal(0, 0.02, 300001).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16).tobytes()
    s = m.lmc_compress(TensorBuffer(raw, ElementType.BF16))
    assert s == O.compress(raw, 1)
    back = m.lmc_decompress(s)
    assert back.data == raw and back.element_type == ElementType.BF16
    for meta, data, stream in load_golden_streams():
        assert m.lmc_decompress(stream).data == data, meta["name"]
    with pytest.raises(UnsupportedFormatError):
        m.lmc_decompress(b"LMC2" + s[4:])
    bad = bytearray(s)
    bad[28 + 16] = 7        # first record's mode byte
    with pytest.raises(CorruptStreamError):
        m.lmc_decompress(bytes(bad))
