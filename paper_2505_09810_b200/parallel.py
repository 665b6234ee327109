"""plmc_compress / plmc_decompress: the reference's data-parallel entry points
(pkg/src/lmc/parallel.py:53-128) on the GPU.

The reference spreads the block-aligned segments of each window over a
process pool; the segment count is a recorded stream property and the worker
count only a scheduling hint, so the stream bytes depend on the input and the
options alone (parallel.py:1-10).  On B200 the unit of parallelism is the
block (one CTA per block, every segment of every window in one launch), so
the worker count has nothing left to schedule: it is validated and otherwise
ignored, and the bytes are those of ``lmc_compress`` with the same options --
exactly the reference's invariant (pkg/tests/test_plmc.py:30-65).
"""
from __future__ import annotations

import os

from .stream import (DEFAULT_BLOCK_SIZE, DEFAULT_BUFFER_SIZE, _WIDTH, _validate_options, lmc_compress,
                     lmc_decompress)
from .types import element_code

# parallel.py:46 -- below this many input bytes the reference encodes in-process.
# Kept for API parity (tests monkeypatch it); output bytes never depend on it.
_MIN_PARALLEL_BYTES = 8 * 1024 * 1024


def _default_workers(segment_count: int) -> int:
    """parallel.py:49-50."""
    return max(1, min(segment_count, os.cpu_count() or 1))


def plmc_compress(buf, *, byte_group: bool = True, block_size: int = DEFAULT_BLOCK_SIZE,
                  segment_count: int | None = None, buffer_size: int = DEFAULT_BUFFER_SIZE,
                  workers: int | None = None) -> bytes:
    """parallel.py:53-103: byte-identical to ``lmc_compress`` with the same
    options; ``segment_count`` defaults to the host's CPU count like the
    reference (it is recorded in the stream), ``workers`` is a hint."""
    if segment_count is None:
        segment_count = os.cpu_count() or 1
    _validate_options(_WIDTH[element_code(buf.element_type)], block_size, segment_count, buffer_size)
    if workers is None:
        workers = _default_workers(segment_count)   # (nothing to schedule: see the module docstring)
    return lmc_compress(buf, byte_group=byte_group, block_size=block_size, segment_count=segment_count,
                        buffer_size=buffer_size)


def plmc_decompress(stream: bytes, worker_count: int | None = None):
    """parallel.py:106-128: decodes any stream with any worker count (every
    segment is decoded concurrently on the device regardless)."""
    return lmc_decompress(stream)
