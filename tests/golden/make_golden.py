"""Generate the golden fixtures from the LIVE reference package (build container only).

Run from the repo root:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference ``lmc`` 0.1.0 from /root/reference/pkg/src (present
only in the build container, never on the GPU box) and writes:

* ``streams.npz``  -- seeded synthetic inputs and the exact streams the
  reference's ``lmc_compress`` produces for them under a spread of options
  (element types, byte-grouping on/off, delta flag, block sizes, segment
  counts, multi-window buffer sizes, empty / tiny / RLE / stored / Huffman /
  package-merge-triggering blocks);
* ``codebooks.npz`` -- histograms and the reference ``build_codebook`` lengths
  (two-queue tie cases, Fibonacci skews that force package-merge, random);
* ``corruptions.json`` -- single-byte mutations of a few reference streams and
  the exception class the reference's ``lmc_decompress`` raises for each
  ("ok" when the mutation decodes), pinning error-class parity.

Inputs are stored, not regenerated, so the fixtures do not depend on numpy's
distribution algorithms staying stable.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

import lmc
from lmc.analysis import bf16_encode
from lmc.entropy import ByteHistogram
from lmc.huffman import build_codebook
from lmc.types import DeltaBuffer, ElementType, TensorBuffer

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_bytes(x: np.ndarray) -> bytes:
    return bf16_encode(x.astype(np.float32)).astype("<u2").tobytes()


def make_inputs(rng: np.random.Generator):
    """(name, bytes, element_type, is_delta, options) cases."""
    cases = []
    # cfg1-like bf16 N(0, .02), plane-aligned (n % 4096 == 0) and misaligned
    x = rng.normal(0, 0.02, 3 * 4096).astype(np.float32)
    cases.append(("bf16_normal_aligned", bf16_bytes(x), ElementType.BF16, False, dict(block_size=4096)))
    x = rng.normal(0, 0.02, 10_007).astype(np.float32)
    cases.append(("bf16_normal_odd", bf16_bytes(x), ElementType.BF16, False, dict(block_size=4096)))
    cases.append(("bf16_normal_odd_seg3", bf16_bytes(x), ElementType.BF16, False, dict(block_size=4096, segment_count=3)))
    cases.append(("bf16_normal_nobg", bf16_bytes(x), ElementType.BF16, False, dict(block_size=4096, byte_group=False)))
    # multi-window: buffer_size not a multiple of block size, windows misaligned
    x = rng.normal(0, 0.02, 40_000).astype(np.float32)
    cases.append(("bf16_multiwindow", bf16_bytes(x), ElementType.BF16, False,
                  dict(block_size=4096, buffer_size=3 * 4096 + 1000, segment_count=2)))
    cases.append(("bf16_multiwindow_64k", bf16_bytes(x), ElementType.BF16, False,
                  dict(block_size=65536, buffer_size=65536 + 2, segment_count=1)))
    # LN-gain-like (1 + N(0, .01)) and bias-like (N(0, .002)) 1-D tensors
    x = 1 + rng.normal(0, 0.01, 768).astype(np.float32)
    cases.append(("bf16_gain_768", bf16_bytes(x), ElementType.BF16, False, {}))
    x = rng.normal(0, 0.002, 3072).astype(np.float32)
    cases.append(("bf16_bias_3072", bf16_bytes(x), ElementType.BF16, False, {}))
    # 50% exact zeros (cfg3a-like) and all zeros (cfg3b-like, RLE)
    x = rng.normal(0, 0.02, 16384).astype(np.float32)
    x[rng.random(16384) < 0.5] = 0.0
    cases.append(("bf16_half_zero", bf16_bytes(x), ElementType.BF16, False, dict(block_size=8192)))
    cases.append(("bf16_zeros", bytes(2 * 20000), ElementType.BF16, False, dict(block_size=4096)))
    # delta of two bf16 steps (cfg4-like): XOR of bit patterns, flag bit1
    w = rng.normal(0, 0.02, 12_000).astype(np.float32)
    w1 = w + rng.normal(0, 1, w.size).astype(np.float32) * (1e-3 * np.abs(w) + 1e-6)
    a, b = np.frombuffer(bf16_bytes(w), np.uint8), np.frombuffer(bf16_bytes(w1), np.uint8)
    cases.append(("bf16_delta", (a ^ b).tobytes(), ElementType.BF16, True, dict(block_size=4096)))
    # fp32 and fp16 4-plane / 2-plane grouping, odd element counts
    x = rng.normal(0, 1, 5003).astype("<f4")
    cases.append(("fp32_normal", x.tobytes(), ElementType.FP32, False, dict(block_size=4096, segment_count=2)))
    x = rng.normal(0, 1, 7001).astype("<f2")
    cases.append(("fp16_normal", x.tobytes(), ElementType.FP16, False, dict(block_size=4096)))
    # raw8: uniform random (stored), skewed (Huffman), tiny, empty
    cases.append(("raw8_random", rng.integers(0, 256, 9000, dtype=np.uint8).tobytes(), ElementType.RAW8, False, dict(block_size=4096)))
    cases.append(("raw8_skewed", (rng.random(20000) ** 3 * 250).astype(np.uint8).tobytes(), ElementType.RAW8, False, dict(block_size=4096, segment_count=16)))
    cases.append(("raw8_one", b"\x07", ElementType.RAW8, False, {}))
    cases.append(("raw8_two", b"\x07\x09", ElementType.RAW8, False, {}))
    cases.append(("raw8_empty", b"", ElementType.RAW8, False, {}))
    cases.append(("bf16_empty", b"", ElementType.BF16, False, {}))
    # package-merge trigger: Fibonacci-distributed symbols in one block
    fib = [1, 1]
    while len(fib) < 26:
        fib.append(fib[-1] + fib[-2])
    syms = np.repeat(np.arange(26, dtype=np.uint8), np.minimum(fib, 40000))
    syms = syms[: 65536]
    rng.shuffle(syms)
    cases.append(("raw8_fibonacci_pm", syms.tobytes(), ElementType.RAW8, False, dict(block_size=65536)))
    # 7-bit fixed-length code (128 equiprobable symbols): Huffman never self-syncs
    cases.append(("raw8_uniform128", rng.integers(0, 128, 8192, dtype=np.uint8).tobytes(), ElementType.RAW8, False, dict(block_size=8192)))
    # two-symbol blocks, near-RLE blocks
    d = np.zeros(6000, dtype=np.uint8)
    d[::997] = 1
    cases.append(("raw8_sparse", d.tobytes(), ElementType.RAW8, False, dict(block_size=4096)))
    return cases


def main() -> None:
    rng = np.random.default_rng(20250510)
    cases = make_inputs(rng)
    meta = []
    inputs, streams = [], []
    for name, data, et, is_delta, opts in cases:
        buf = DeltaBuffer(data, et, 0, 1) if is_delta else TensorBuffer(data, et)
        stream = lmc.lmc_compress(buf, **opts)
        assert lmc.lmc_decompress(stream).data == data
        full = dict(byte_group=True, block_size=65536, segment_count=1, buffer_size=128 << 20)
        full.update(opts)
        meta.append(dict(name=name, element_type=et.code, delta=is_delta, **full,
                         input_len=len(data), stream_len=len(stream)))
        inputs.append(np.frombuffer(data, np.uint8))
        streams.append(np.frombuffer(stream, np.uint8))
    np.savez_compressed(
        os.path.join(HERE, "streams.npz"),
        meta=np.array(json.dumps(meta)),
        inputs=np.concatenate(inputs) if inputs else np.zeros(0, np.uint8),
        streams=np.concatenate(streams),
    )

    # codebooks
    hists, lens = [], []

    def add(c):
        c = np.asarray(c, dtype=np.int64)
        full = np.zeros(256, dtype=np.int64)
        full[: c.size] = c
        if full.sum() == 0:
            return
        hists.append(full)
        lens.append(build_codebook(ByteHistogram(full, int(full.sum()))).lengths.copy())

    add([5, 2, 1, 1])
    add([1, 1, 2, 2])
    add([7])
    add(np.ones(256))
    for k in range(2, 40):
        fib = [1, 1]
        while len(fib) < k:
            fib.append(fib[-1] + fib[-2])
        add(fib[:k])
    for t in range(1500):
        k = int(rng.integers(2, 257))
        kind = t % 4
        if kind == 0:
            c = rng.integers(1, 100, k)
        elif kind == 1:
            c = (rng.random(k) ** 8 * 1e5).astype(int) + 1
        elif kind == 2:
            c = np.floor(np.exp(rng.normal(0, 4, k))).astype(int) + 1
            c = np.minimum(c, 1 << 20)
        else:
            fib = [1, 1]
            while len(fib) < k:
                fib.append(min(fib[-1] + fib[-2], 1 << 20))
            c = np.array(fib[:k]) + rng.integers(0, 3, k)
        full = np.zeros(256, dtype=np.int64)
        full[rng.choice(256, k, replace=False)] = c
        add(full)
    np.savez_compressed(os.path.join(HERE, "codebooks.npz"), hists=np.stack(hists).astype(np.uint32), lengths=np.stack(lens))

    # corruption classes
    corr = []
    by_name = {m["name"]: i for i, m in enumerate(meta)}
    offs = np.concatenate([[0], np.cumsum([s.size for s in streams])])
    for name in ("bf16_normal_odd_seg3", "raw8_skewed", "bf16_multiwindow", "bf16_zeros", "raw8_one"):
        i = by_name[name]
        s = streams[i].tobytes()
        positions = sorted(set(list(range(0, len(s), max(1, len(s) // 60))) + list(range(0, min(len(s), 40)))))
        for pos in positions:
            val = int(rng.integers(1, 256))
            bad = bytearray(s)
            bad[pos] ^= val
            try:
                out = lmc.lmc_decompress(bytes(bad))
                res = "ok" if out.data == inputs[i].tobytes() else "ok_changed"
            except lmc.LmcError as exc:
                res = type(exc).__name__
            corr.append(dict(case=name, kind="xor", pos=pos, val=val, result=res))
        for cut in sorted(set([len(s) - 1, len(s) // 2, 28 + 3, 10, 0])):
            if cut >= len(s):
                continue
            try:
                lmc.lmc_decompress(s[:cut])
                res = "ok"
            except lmc.LmcError as exc:
                res = type(exc).__name__
            corr.append(dict(case=name, kind="truncate", pos=cut, val=0, result=res))
        try:
            lmc.lmc_decompress(s + b"\x00")
            res = "ok"
        except lmc.LmcError as exc:
            res = type(exc).__name__
        corr.append(dict(case=name, kind="append", pos=len(s), val=0, result=res))
    with open(os.path.join(HERE, "corruptions.json"), "w") as f:
        json.dump(corr, f, indent=0)
    print(f"{len(meta)} streams, {len(hists)} codebooks, {len(corr)} corruptions", file=sys.stderr)


if __name__ == "__main__":
    main()
