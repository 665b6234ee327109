"""Multi-GPU sharding of a checkpoint: one process per GPU, whole tensors per rank.

The reference's data parallelism is a CPU process pool over block-aligned
segments of ONE stream (pkg/src/lmc/parallel.py:53-128); its callers hand it
one tensor at a time (chain.py:187, cli.py:155).  A checkpoint is many
independent streams, one per tensor, so on B200 the natural unit of
distribution is the tensor: each rank compresses the tensors it owns with no
data-path collective, and the only exchange is an all-gather of the
per-stream compressed sizes, from which every rank derives the same manifest
(stream offsets in the packed checkpoint file).  Each rank then writes its own
streams at their final offsets; the packed file is byte-identical to the one
a single GPU (or the reference, stream by stream) produces.

Assignment is greedy largest-first bin packing on uncompressed bytes
(deterministic: ties in size by tensor index, ties in load by rank index), so
every rank computes the same owner table without communicating.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np


def assign_tensors(nbytes: Sequence[int], world: int) -> list[int]:
    """Owner rank of every tensor (largest first onto the least-loaded rank)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    order = sorted(range(len(nbytes)), key=lambda i: (-int(nbytes[i]), i))
    load = [0] * world
    owner = [0] * len(nbytes)
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[i] = r
        load[r] += int(nbytes[i])
    return owner


def manifest_offsets(lengths: Sequence[int], base: int = 0) -> list[int]:
    """Start of every stream in the packed checkpoint (streams back to back)."""
    out, pos = [], base
    for n in lengths:
        out.append(pos)
        pos += int(n)
    return out


def gather_lengths(local: dict[int, int], n: int, group=None, device=None) -> list[int]:
    """All-gather the compressed length of every stream from its owner.

    ``local`` maps the stream indices this rank owns to their lengths.  One
    collective per checkpoint: every rank contributes an n-vector (zeros where
    it is not the owner) and the gathered rows are summed.
    """
    import torch
    import torch.distributed as dist

    vec = torch.zeros(n, dtype=torch.int64, device=device)
    for i, v in local.items():
        vec[i] = int(v)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [int(x) for x in vec.tolist()]
    ws = dist.get_world_size(group)
    rows = torch.empty(ws * n, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(rows, vec, group=group)
    return [int(x) for x in rows.view(ws, n).sum(0).tolist()]


@dataclass
class ShardResult:
    """One rank's share of a sharded compress."""

    rank: int
    world: int
    owner: list[int]                 # owner rank of every tensor
    owned: list[int]                 # indices this rank compressed
    streams: dict[int, bytes]        # owned index -> LMC1 stream
    lengths: list[int]               # every stream's length (all ranks)
    offsets: list[int]               # every stream's offset in the packed file

    @property
    def total_bytes(self) -> int:
        return (self.offsets[-1] + self.lengths[-1]) if self.lengths else 0

    def write_into(self, fd: int) -> None:
        """pwrite this rank's streams at their manifest offsets (shared file)."""
        for i in self.owned:
            os.pwrite(fd, self.streams[i], self.offsets[i])

    def manifest(self) -> list[dict]:
        return [{"index": i, "offset": o, "length": n, "rank": r}
                for i, (o, n, r) in enumerate(zip(self.offsets, self.lengths, self.owner))]


def compress_sharded(tensors: Sequence, *, nbytes: Sequence[int] | None = None, group=None,
                     compress_fn: Callable | None = None, collective_device=None, **options) -> ShardResult:
    """Compress a checkpoint across the ranks of ``group``.

    ``tensors[i]`` only needs to be valid on the rank that owns tensor i
    (other entries may be None if ``nbytes`` gives the sizes).  By default the
    owned tensors are compressed in ONE batched GPU call
    (``stream.compress_many``); ``compress_fn(list_of_owned) -> list[bytes]``
    replaces that call (tests use it to exercise the sharding logic on CPU).
    """
    import torch.distributed as dist

    if dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    if nbytes is None:
        nbytes = [_nbytes(t) for t in tensors]
    owner = assign_tensors(nbytes, world)
    owned = [i for i, r in enumerate(owner) if r == rank]
    if compress_fn is None:
        from .stream import compress_many

        compress_fn = lambda bufs: compress_many(bufs, **options)  # noqa: E731
    outs = compress_fn([tensors[i] for i in owned]) if owned else []
    streams = {i: bytes(s) for i, s in zip(owned, outs)}
    lengths = gather_lengths({i: len(s) for i, s in streams.items()}, len(nbytes), group=group,
                             device=collective_device)
    return ShardResult(rank, world, owner, owned, streams, lengths, manifest_offsets(lengths))


def decompress_sharded(packed, lengths: Sequence[int], owner: Sequence[int], *, rank: int,
                       decompress_fn: Callable | None = None) -> dict[int, object]:
    """Decode the streams this rank owns out of a packed checkpoint."""
    offs = manifest_offsets(lengths)
    mine = [i for i, r in enumerate(owner) if r == rank]
    view = memoryview(packed)
    streams = [bytes(view[offs[i]:offs[i] + lengths[i]]) for i in mine]
    if decompress_fn is None:
        from .stream import decompress_many

        decompress_fn = decompress_many
    return dict(zip(mine, decompress_fn(streams))) if mine else {}


def _nbytes(t) -> int:
    if t is None:
        raise ValueError("tensor sizes are needed for unowned entries: pass nbytes=")
    if hasattr(t, "data") and isinstance(t.data, (bytes, bytearray, memoryview)):
        return len(t.data)        # TensorBuffer / DeltaBuffer (types.py)
    if hasattr(t, "numel"):
        return int(t.numel() * t.element_size())
    return int(np.asarray(t).nbytes)
