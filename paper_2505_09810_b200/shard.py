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


# ------------------------------------------------- splitting one tensor
# A tensor larger than a rank's fair share is split by block range (SURVEY
# §8(e)): rank r compresses blocks [b_r, b_{r+1}) of the stream's record list
# and the raw CRC-32 of payload bytes [c_r, c_{r+1}) (Codec.compress_part /
# lmcg_compress_part); one all-gather of record sizes and CRCs lets every
# rank place its records, and the header (CRC combined) and segment tables
# are written from the gathered sizes (stream.py:100-111, 271-284, 344-355).

_P = 0xEDB88320


def _multmodp(a: int, b: int) -> int:
    m, p = 1 << 31, 0
    while m:
        if a & m:
            p ^= b
            if (a & (m - 1)) == 0:
                break
        m >>= 1
        b = (b >> 1) ^ _P if b & 1 else b >> 1
    return p


def crc_shift(c: int, nbytes: int) -> int:
    """Raw CRC-32 c followed by nbytes zero bytes (GF(2) x^(8n) mod P)."""
    x2n = 1 << 30   # x^1
    p = 1 << 31     # x^0
    n, k = nbytes, 0
    xk = x2n
    # x^(2^k) for k = 3.. (8 n = n << 3)
    for _ in range(3):
        xk = _multmodp(xk, xk)
    while n:
        if n & 1:
            p = _multmodp(xk, p)
        n >>= 1
        xk = _multmodp(xk, xk)
    return _multmodp(p, c) if c else 0


def crc_combine(parts: Sequence[tuple[int, int]]) -> int:
    """zlib.crc32 of the concatenation of byte ranges given as (raw CRC, length)."""
    raw, total = 0, 0
    for c, n in parts:
        raw = crc_shift(raw, n) ^ c
        total += n
    return raw ^ crc_shift(0xFFFFFFFF, total) ^ 0xFFFFFFFF


def stream_layout(nbytes: int, width: int, byte_group: bool, block_size: int, segment_count: int,
                  buffer_size: int) -> list[dict]:
    """Windows of a stream: bytes, first block, block count and, per segment,
    (original bytes, first block, end block) -- the record order of the stream."""
    from .stream import segment_bounds

    out, blk = [], 0
    for woff in range(0, nbytes, buffer_size):
        W = min(buffer_size, nbytes - woff)
        nb = (W + block_size - 1) // block_size
        segs = []
        for ea, eb in segment_bounds(W, block_size, segment_count):
            ba = ea // block_size
            bb = ba if eb == ea else (eb + block_size - 1) // block_size
            segs.append((eb - ea, blk + ba, blk + bb))
        out.append({"W": W, "blk0": blk, "nblocks": nb, "segments": segs})
        blk += nb
    return out


def split_ranges(nblocks: int, nbytes: int, world: int) -> list[tuple[int, int, int, int]]:
    """Balanced (block range, CRC byte range) of every rank."""
    return [(nblocks * r // world, nblocks * (r + 1) // world, nbytes * r // world, nbytes * (r + 1) // world)
            for r in range(world)]


def assemble_stream(nbytes: int, element_type: int, flags: int, block_size: int, segment_count: int,
                    buffer_size: int, rec_sizes: Sequence[int], records: bytes,
                    crc_parts: Sequence[tuple[int, int]]) -> bytes:
    """The LMC1 stream from all records (in record order, back to back), their
    sizes and the (raw CRC, length) of consecutive payload byte ranges."""
    import struct

    from .stream import _WIDTH

    lay = stream_layout(nbytes, _WIDTH[element_type], bool(flags & 1), block_size, segment_count, buffer_size)
    offs = [0]
    for n in rec_sizes:
        offs.append(offs[-1] + int(n))
    crc = crc_combine(crc_parts) if nbytes else 0
    out = [struct.pack("<4sBBBBQIII", b"LMC1", 1, flags, element_type, 0, nbytes, block_size, segment_count, crc)]
    for w in lay:
        tab = b"".join(struct.pack("<QQ", orig, offs[bb] - offs[ba]) for orig, ba, bb in w["segments"])
        out.append(tab)
        out.append(records[offs[w["blk0"]]:offs[w["blk0"] + w["nblocks"]]])
    return b"".join(out)


def compress_split(tensor, *, group=None, element_type: int | None = None, prev=None, byte_group: bool = True,
                   block_size: int = 65536, segment_count: int = 1, buffer_size: int = 128 << 20,
                   codec=None, part_fn: Callable | None = None):
    """Compress ONE tensor with all ranks of ``group`` (each holds the whole
    tensor, e.g. replicated parameters): rank r compresses its block range,
    one all-gather exchanges record sizes / CRCs / parts, and every rank
    returns the full stream (byte-identical to a one-GPU lmc_compress).

    ``part_fn(blk_a, blk_b, crc_a, crc_b) -> (records: bytes, sizes: list,
    raw_crc: int)`` replaces the GPU part compression (tests drive the
    exchange logic on CPU with it)."""
    import torch.distributed as dist

    from .stream import _WIDTH, _bytes_view, _torch_et

    if dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    et = int(element_type if element_type is not None else _torch_et(tensor.dtype))
    nbytes = int(_bytes_view(tensor).numel()) if hasattr(tensor, "data_ptr") else len(tensor)
    lay = stream_layout(nbytes, _WIDTH[et], byte_group, block_size, segment_count, buffer_size)
    nblk = sum(w["nblocks"] for w in lay)
    ranges = split_ranges(nblk, nbytes, world)
    ba, bb, ca, cb = ranges[rank]
    if part_fn is None:
        codec = codec or __import__("paper_2505_09810_b200").stream.default_codec()
        rec, sizes, crc = codec.compress_part(tensor, ba, bb, ca, cb, element_type=et, prev=prev, byte_group=byte_group,
                                              block_size=block_size, segment_count=segment_count,
                                              buffer_size=buffer_size)
        sizes = [int(x) for x in sizes.tolist()]
        records = rec[:sum(sizes)].cpu().numpy().tobytes()
        raw = int(crc.item()) & 0xFFFFFFFF
    else:
        records, sizes, raw = part_fn(ba, bb, ca, cb)
    flags = (1 if byte_group else 0) | (2 if prev is not None else 0)
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (sizes, raw, records), group=group)
    else:
        gathered = [(sizes, raw, records)]
    all_sizes = [x for g in gathered for x in g[0]]
    crc_parts = [(g[1], ranges[r][3] - ranges[r][2]) for r, g in enumerate(gathered)]
    return assemble_stream(nbytes, et, flags, block_size, segment_count, buffer_size, all_sizes,
                           b"".join(g[2] for g in gathered), crc_parts)


def _nbytes(t) -> int:
    if t is None:
        raise ValueError("tensor sizes are needed for unowned entries: pass nbytes=")
    if hasattr(t, "data") and isinstance(t.data, (bytes, bytearray, memoryview)):
        return len(t.data)        # TensorBuffer / DeltaBuffer (types.py)
    if hasattr(t, "numel"):
        return int(t.numel() * t.element_size())
    return int(np.asarray(t).nbytes)
