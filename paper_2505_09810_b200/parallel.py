"""Data-parallel entry points, mirroring the reference's PLMC driver
(pkg/src/lmc/parallel.py:53-128).

On the CPU the reference farms block-aligned segments out to a process pool;
here the data parallelism is the GPU grid (one CTA per block), so ``workers``
/ ``worker_count`` are accepted for signature compatibility and ignored.
``segment_count`` keeps its stream-format meaning (it is recorded in the
header), and defaults to ``os.cpu_count()`` exactly like the reference, so
plmc streams are byte-identical to the reference's on the same machine
options.
"""
from __future__ import annotations

import os

from .stream import DEFAULT_BLOCK_SIZE, DEFAULT_BUFFER_SIZE, lmc_compress, lmc_decompress


def plmc_compress(buf, *, byte_group: bool = True, block_size: int = DEFAULT_BLOCK_SIZE,
                  segment_count: int | None = None, buffer_size: int = DEFAULT_BUFFER_SIZE,
                  workers: int | None = None) -> bytes:
    if segment_count is None:
        segment_count = os.cpu_count() or 1
    return lmc_compress(buf, byte_group=byte_group, block_size=block_size, segment_count=segment_count,
                        buffer_size=buffer_size)


def plmc_decompress(stream: bytes, worker_count: int | None = None):
    return lmc_decompress(stream)
