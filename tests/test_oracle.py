"""Pin the C oracle (oracle/lmc_oracle.c) against the reference.

Every test here runs on CPU.  The golden fixtures were produced by the live
reference (tests/golden/make_golden.py); the known-answer values restate the
reference's own unit tests (pkg/tests/test_huffman.py, test_stream.py,
test_bytegroup.py, golden/meta.json).
"""
import numpy as np
import pytest

from conftest import (load_golden_codebooks, load_golden_corruptions,
                      load_golden_streams, reference_lmc)
from oracle import oracle as O

CLASS = {"CorruptStreamError": O.CORRUPT, "IntegrityError": O.INTEGRITY,
         "UnsupportedFormatError": O.UNSUPPORTED}


@pytest.mark.parametrize("case", load_golden_streams(), ids=lambda c: c[0]["name"])
def test_oracle_reproduces_reference_streams(case):
    m, data, stream = case
    got = O.compress(data, m["element_type"], delta=m["delta"], byte_group=m["byte_group"],
                     block_size=m["block_size"], segment_count=m["segment_count"],
                     buffer_size=m["buffer_size"], threads=2)
    assert got == stream
    out, et, flags = O.decompress(stream, threads=2)
    assert out == data and et == m["element_type"]
    assert flags == (int(m["byte_group"]) | (2 if m["delta"] else 0))


def test_oracle_codebooks_match_reference():
    hists, lengths = load_golden_codebooks()
    npm = 0
    for h, want in zip(hists, lengths):
        got, pm = O.build_codebook(h.astype(np.uint64))
        npm += pm
        assert (got == want).all()
    assert npm > 50  # package-merge path is exercised


def test_oracle_corruption_classes_match_reference():
    streams = {m["name"]: (d, s) for m, d, s in load_golden_streams()}
    for c in load_golden_corruptions():
        data, s = streams[c["case"]]
        if c["kind"] == "xor":
            bad = bytearray(s)
            bad[c["pos"]] ^= c["val"]
        elif c["kind"] == "truncate":
            bad = s[: c["pos"]]
        else:
            bad = s + b"\x00"
        try:
            out, _, _ = O.decompress(bytes(bad))
            res = "ok"
            assert out == data
        except O.OracleError as exc:
            res = exc.code
        want = c["result"] if c["result"] == "ok" else CLASS[c["result"]]
        assert res == want, c


# --- known answers restated from the reference's unit tests ----------------

def test_known_lengths_5211():  # test_huffman.py:46-52
    h = np.zeros(256, np.uint64); h[:4] = [5, 2, 1, 1]
    assert list(O.build_codebook(h)[0][:4]) == [1, 2, 3, 3]


def test_leaf_first_ties():  # [1,1,2,2] -> (2,2,2,2)
    h = np.zeros(256, np.uint64); h[:4] = [1, 1, 2, 2]
    assert list(O.build_codebook(h)[0][:4]) == [2, 2, 2, 2]


def test_uniform_256_all_eight():  # test_huffman.py:59-61
    assert (O.build_codebook(np.ones(256, np.uint64))[0] == 8).all()


def test_fibonacci_hits_limit():  # test_huffman.py:76-86
    fib = [1, 1]
    while len(fib) < 30:
        fib.append(fib[-1] + fib[-2])
    h = np.zeros(256, np.uint64); h[:30] = fib
    lens, pm = O.build_codebook(h)
    assert pm and lens.max() == 15
    assert sum(2.0 ** -int(l) for l in lens if l) == 1.0


def test_abab_encoding():  # test_huffman.py:200-207 (lengths A=1, B=2, underfull code)
    lens = np.zeros(256, np.uint8); lens[ord("A")] = 1; lens[ord("B")] = 2
    data, bits = O.encode_block(b"ABAB", lens)
    assert data == b"\x48" and bits == 6
    assert O.decode_block(b"\x48", 6, lens, 4) == b"ABAB"


def test_group_bytes_layouts():  # test_bytegroup.py:11-29 (SPEC examples)
    assert O.group_bytes(bytes([2, 1, 4, 3, 6, 5, 8, 7]), 2) == bytes([2, 4, 6, 8, 1, 3, 5, 7])
    assert O.group_bytes(bytes([1, 2, 3, 4, 5, 6, 7, 8]), 4) == bytes([1, 5, 2, 6, 3, 7, 4, 8])


def test_zeros_bf16_known_answer():  # golden/meta.json:13-23
    s = O.compress(bytes(8192), 1, block_size=4096)
    assert len(s) == 56
    assert O.crc32(bytes(8192)) == 3639908756


def test_rle_and_stored_record_sizes(rng):  # test_stream.py:37-48
    s = O.compress(bytes(65536), 0, byte_group=False)
    assert len(s) == 28 + 16 + 6
    r = rng.integers(0, 256, 65536, dtype=np.uint8).tobytes()
    s = O.compress(r, 0, byte_group=False)
    assert len(s) == 28 + 16 + 65536 + 5


def test_empty_input_is_header_only():  # test_stream.py:198-203
    for et in range(4):
        s = O.compress(b"", et)
        assert len(s) == 28
        assert O.decompress(s)[0] == b""


def test_text_raw8_known_answer():  # golden/meta.json:2-12 (fixture only in the build container)
    import os
    p = "/root/reference/pkg/tests/golden/text_raw8.bin"
    if not os.path.exists(p):
        pytest.skip("reference fixture not present")
    data = open(p, "rb").read()
    s = O.compress(data, 0, byte_group=False, block_size=4096)
    assert len(s) == 3430 and O.crc32(data) == 3773586408


def test_live_reference_differential(rng):
    lmc = reference_lmc()
    if lmc is None:
        pytest.skip("live reference not importable here")
    from lmc.types import ElementType, TensorBuffer
    for trial in range(6):
        n = int(rng.integers(0, 300_000))
        et = list(ElementType)[trial % 4]
        n -= n % et.width
        d = (rng.random(n) ** (1 + trial) * 255).astype(np.uint8).tobytes()
        opts = dict(block_size=int(2 ** rng.integers(12, 17)), segment_count=int(rng.integers(1, 6)),
                    byte_group=bool(trial % 2 == 0))
        opts["buffer_size"] = int(opts["block_size"] * rng.integers(1, 5) + et.width * rng.integers(0, 50))
        want = lmc.lmc_compress(TensorBuffer(d, et), **opts)
        got = O.compress(d, et.value[0], threads=3, **opts)
        assert got == want
