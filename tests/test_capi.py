"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/lmc_b200.h declares, and the host-side mirror logic matches
the reference (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden_streams

import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import _build, _lib
from oracle import oracle as O


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lmc_b200.h")).read()
    return sorted(set(re.findall(r"\b(lmcg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert syms == sorted(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    so = _build.build()
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_validate_options_matches_reference_rules(lib):
    def v(bs, segs, buf, et=1, n=0):
        o = _lib.lmcg_options(1, bs, segs, 0, buf)
        return lib.lmcg_validate_options(ctypes.byref(o), et, n)

    assert v(65536, 1, 128 << 20) == 0
    assert v(1000, 1, 1 << 20) == 4          # not a power of two
    assert v(2048, 1, 1 << 20) == 4          # below 4 KiB
    assert v(1 << 21, 1, 1 << 22) == 4       # above 1 MiB
    assert v(4096, 0, 1 << 20) == 4          # segments < 1
    assert v(4096, 1, 1024) == 4             # buffer < block
    assert v(4096, 1, 4096 + 2, et=3) == 4   # buffer not element aligned
    assert v(4096, 1, 8192, et=3, n=6) == 5  # payload not element aligned


def test_compress_bound_matches_oracle(lib):
    for n, bs, segs, buf in [(0, 4096, 1, 8192), (1, 4096, 3, 4096), (300_001, 4096, 1, 128 << 20),
                             (10_000_000, 65536, 8, 3 << 20)]:
        t = _lib.lmcg_tensor(None, None, n, 0, 0)
        o = _lib.lmcg_options(1, bs, segs, 0, buf)
        assert lib.lmcg_compress_bound(ctypes.byref(t), 1, ctypes.byref(o)) == O.lib().lmco_compress_bound(n, bs, segs, buf)


def test_parse_header_and_segment_bounds_host_logic():
    for m, data, stream in load_golden_streams():
        h = lmcb.parse_header(stream)
        assert h.original_length == len(data) and h.block_size == m["block_size"]
        assert h.segment_count == m["segment_count"] and h.byte_grouped == m["byte_group"]
        assert h.delta_applied == m["delta"]
        assert h.pack() == stream[:28]
    b = lmcb.segment_bounds(5000, 4096, 8)
    assert len(b) == 8 and sum(y - x for x, y in b) == 5000 and sum(1 for x, y in b if x == y) == 6
    with pytest.raises(lmcb.UnsupportedFormatError):
        lmcb.parse_header(b"LMC1")
    with pytest.raises(lmcb.CorruptStreamError):
        lmcb.parse_header(b"LMC1\x01\x84" + bytes(22))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lmcb.DeviceError):
        lmcb.lmc_compress(lmcb.TensorBuffer(b"abcd", lmcb.ElementType.RAW8))
    with pytest.raises(lmcb.DeviceError):
        lmcb.lmc_decompress(b"LMC1")


def test_error_classes_mirror_reference():
    for name in ["LmcError", "AlignmentError", "ShapeMismatchError", "DtypeMismatchError", "EmptyInputError",
                 "MalformedCodebookError", "MissingSymbolError", "CorruptStreamError", "UnsupportedFormatError",
                 "IntegrityError", "ConfigError"]:
        cls = getattr(lmcb, name)
        assert issubclass(cls, lmcb.LmcError)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2505_09810_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("oracle/", ""), f
