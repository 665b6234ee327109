"""Padding bits after the last codeword of a Huffman record are not checked by
the reference (huffman.py:338-348 checks only the end position, and the CRC
covers the decoded payload), so a stream whose last record has a flipped
padding bit must still decode, with the same payload and no error
(SURVEY App. A).  A flipped bit inside the codewords must not decode silently."""
import struct

import numpy as np
import pytest

from oracle import oracle as O

BF16 = 1


def _stream_with_padding():
    """A bf16 stream of two 64 KiB blocks (low plane stored, high plane
    Huffman) whose Huffman record leaves >= 1 padding bit in its last byte."""
    for seed in range(50):
        rng = np.random.default_rng(seed)
        w = rng.normal(0, 0.02, 65536).astype(np.float32)
        raw = (w.view(np.uint32) >> 16).astype(np.uint16).tobytes()
        s = O.compress(raw, BF16)
        # header 28 | segment table 16 | stored record 5 + 65536 | huffman record
        pos = 28 + 16 + 5 + 65536
        assert s[28 + 16] == 2 and s[pos] == 0
        bits = struct.unpack_from("<I", s, pos + 5 + 128)[0]
        assert len(s) == pos + 5 + 132 + (bits + 7) // 8
        if bits % 8:
            return raw, s, bits
    raise AssertionError("no seed with padding bits")


def _flip_padding(s, bits):
    b = bytearray(s)
    pad = 8 - bits % 8
    b[-1] ^= 1 << (pad - 1)          # the first padding bit (MSB-first packing)
    return bytes(b)


def test_oracle_accepts_flipped_padding_bit():
    raw, s, bits = _stream_with_padding()
    bad = _flip_padding(s, bits)
    assert bad != s
    out, et, flags = O.decompress(bad)
    assert out == raw and et == BF16
    # and a codeword bit is not padding: the oracle rejects that flip
    b = bytearray(s)
    b[-1] ^= 0x80
    with pytest.raises(O.OracleError):
        O.decompress(bytes(b))


@pytest.mark.gpu
def test_gpu_accepts_flipped_padding_bit():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_09810_b200 as lmcb

    raw, s, bits = _stream_with_padding()
    bad = _flip_padding(s, bits)
    # the GPU writes the same stream, and decodes both
    from paper_2505_09810_b200.types import ElementType, TensorBuffer
    assert lmcb.lmc_compress(TensorBuffer(raw, ElementType.BF16)) == s
    assert lmcb.lmc_decompress(bad).data == raw
    codec = lmcb.Codec()
    dev = torch.frombuffer(bytearray(bad), dtype=torch.uint8).cuda()
    codec.ctx.lib.lmcg_fallback_segments(1)
    r = codec.decompress([dev])
    assert r.status == [0]
    assert bytes(r.payload(0).cpu().numpy()) == raw


@pytest.mark.gpu
def test_gpu_rejects_flipped_codeword_bit():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_09810_b200 as lmcb
    from paper_2505_09810_b200.errors import IntegrityError

    raw, s, bits = _stream_with_padding()
    b = bytearray(s)
    b[-1] ^= 0x80                    # first bit of the last byte: a codeword bit
    # the reference decodes other symbols here and reports the CRC mismatch
    # (checked against lmc.lmc_decompress when this test was written)
    with pytest.raises(IntegrityError):
        lmcb.lmc_decompress(bytes(b))
