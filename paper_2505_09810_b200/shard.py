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


def collective_device(group=None, device=None):
    """Device of the exchange tensors: ``device`` if given, else the current
    CUDA device under an NCCL group (NCCL moves device tensors only) and the
    CPU otherwise (gloo)."""
    import torch
    import torch.distributed as dist

    if device is not None:
        return torch.device(device)
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_lengths(local: dict[int, int], n: int, group=None, device=None) -> list[int]:
    """All-gather the compressed length of every stream from its owner.

    ``local`` maps the stream indices this rank owns to their lengths.  One
    collective per checkpoint: every rank contributes an n-vector (zeros where
    it is not the owner) and the gathered rows are summed.  The vectors live
    on ``collective_device(group, device)`` (CUDA under NCCL).
    """
    import torch
    import torch.distributed as dist

    dev = collective_device(group, device)
    host = torch.zeros(n, dtype=torch.int64)
    for i, v in local.items():
        host[i] = int(v)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [int(x) for x in host.tolist()]
    vec = host.to(dev)
    ws = dist.get_world_size(group)
    rows = torch.empty(ws * n, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(rows, vec, group=group)
    return [int(x) for x in rows.view(ws, n).sum(0).tolist()]


def gather_device_lengths(lengths, owned: Sequence[int], n: int, group=None):
    """Device variant: ``lengths`` (int64 CUDA tensor, one per owned stream, in
    ``owned`` order) scattered into an n-vector and all-gathered over the
    group without a host round trip.  Returns the summed n-vector (device)."""
    import torch
    import torch.distributed as dist

    dev = lengths.device
    vec = torch.zeros(n, dtype=torch.int64, device=dev)
    if len(owned):
        vec.index_copy_(0, torch.as_tensor(list(owned), dtype=torch.int64, device=dev), lengths.to(torch.int64))
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return vec
    ws = dist.get_world_size(group)
    rows = torch.empty(ws * n, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(rows, vec, group=group)
    return rows.view(ws, n).sum(0)


def _pwrite_all(fd: int, data, offset: int) -> None:
    """os.pwrite until every byte is written (one call moves at most ~2 GiB)."""
    view = memoryview(data).cast("B")
    while len(view):
        k = os.pwrite(fd, view, offset)
        if k <= 0:
            raise OSError(f"pwrite wrote {k} bytes at offset {offset}")
        view = view[k:]
        offset += k


@dataclass
class ShardResult:
    """One rank's share of a sharded compress.

    The owned streams are either host bytes (``streams``) or, for CUDA
    inputs, still in HBM (``batch``: a CompressedBatch whose stream k is
    ``owned[k]``); ``stream_bytes(i)`` copies one to the host on demand."""

    rank: int
    world: int
    owner: list[int]                 # owner rank of every tensor
    owned: list[int]                 # indices this rank compressed
    streams: dict[int, bytes]        # owned index -> LMC1 stream (host results)
    lengths: list[int]               # every stream's length (all ranks)
    offsets: list[int]               # every stream's offset in the packed file
    batch: object = None             # device CompressedBatch of the owned streams (CUDA inputs)

    @property
    def total_bytes(self) -> int:
        return (self.offsets[-1] + self.lengths[-1]) if self.lengths else 0

    def stream_bytes(self, i: int) -> bytes:
        if i in self.streams:
            return self.streams[i]
        k = self.owned.index(i)
        return self.batch.stream(k).cpu().numpy().tobytes()

    def write_into(self, fd: int) -> None:
        """pwrite this rank's streams at their manifest offsets (shared file)."""
        if self.batch is not None and self.owned:
            # one device->host copy of the rank's packed streams, then a write
            # per stream at its manifest offset
            off, ln = self.batch.host_layout()
            host = self.batch.data[: off[-1] + ln[-1]].cpu().numpy()
            for k, i in enumerate(self.owned):
                _pwrite_all(fd, host[off[k]: off[k] + ln[k]], self.offsets[i])
            return
        for i in self.owned:
            _pwrite_all(fd, self.streams[i], self.offsets[i])

    def manifest(self) -> list[dict]:
        return [{"index": i, "offset": o, "length": n, "rank": r}
                for i, (o, n, r) in enumerate(zip(self.offsets, self.lengths, self.owner))]


def _is_cuda(t) -> bool:
    return hasattr(t, "is_cuda") and bool(t.is_cuda)


def compress_sharded(tensors: Sequence, *, nbytes: Sequence[int] | None = None, group=None,
                     compress_fn: Callable | None = None, collective_device=None, codec=None,
                     prev: Sequence | None = None, **options) -> ShardResult:
    """Compress a checkpoint across the ranks of ``group``.

    ``tensors[i]`` only needs to be valid on the rank that owns tensor i
    (other entries may be None if ``nbytes`` gives the sizes).  CUDA tensors
    are compressed in ONE batched device call (``Codec.compress``; with
    ``prev``, against the previous step, fused XOR) and their streams stay in
    HBM; host buffers (TensorBuffer / DeltaBuffer) go through
    ``stream.compress_many``.  ``compress_fn(list_of_owned) -> list[bytes]``
    replaces either (tests use it to exercise the sharding logic on CPU).
    The only exchange is the all-gather of the stream lengths.
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
    batch = None
    streams: dict[int, bytes] = {}
    if compress_fn is None and owned and all(_is_cuda(tensors[i]) for i in owned):
        from .stream import default_codec

        codec = codec or default_codec()
        pv = None if prev is None else [prev[i] for i in owned]
        batch = codec.compress([tensors[i] for i in owned], prev=pv, **options)
        _, ln = batch.host_layout()
        local = dict(zip(owned, ln))
    else:
        if compress_fn is None:
            from .stream import compress_many

            compress_fn = lambda bufs: compress_many(bufs, **options)  # noqa: E731
        outs = compress_fn([tensors[i] for i in owned]) if owned else []
        streams = {i: bytes(s) for i, s in zip(owned, outs)}
        local = {i: len(s) for i, s in streams.items()}
    lengths = gather_lengths(local, len(nbytes), group=group, device=collective_device)
    return ShardResult(rank, world, owner, owned, streams, lengths, manifest_offsets(lengths), batch)


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


@dataclass
class SplitStream:
    """One rank's part of ONE stream compressed by all ranks (compress_split).

    Every rank knows the whole stream's layout (header, segment tables and
    the offset of every record) from the gathered record sizes; it holds only
    its own records.  ``write_into`` places them in a shared file (rank 0
    also writes the header and the segment tables); ``to_bytes`` gathers the
    whole stream (moving every rank's records: a convenience, not the data
    path)."""

    rank: int
    world: int
    length: int                                   # bytes of the whole stream
    frame: list[tuple[int, bytes]]                # (offset, bytes): header + segment tables
    pieces: list[tuple[int, int, int]]            # (stream offset, local offset, bytes) of local records
    records: object                               # this rank's records, back to back (bytes or CUDA tensor)
    group: object = None

    def _local(self) -> bytes:
        r = self.records
        return bytes(r) if isinstance(r, (bytes, bytearray)) else r.cpu().numpy().tobytes()

    def write_into(self, fd: int, base: int = 0) -> None:
        if self.rank == 0:
            for off, b in self.frame:
                _pwrite_all(fd, b, base + off)
        loc = memoryview(self._local())
        for so, lo, n in self.pieces:
            _pwrite_all(fd, loc[lo: lo + n], base + so)

    def to_bytes(self) -> bytes:
        import torch
        import torch.distributed as dist

        out = bytearray(self.length)
        for off, b in self.frame:
            out[off: off + len(b)] = b
        if self.world == 1:
            parts = [(self.pieces, self._local())]
        else:
            dev = collective_device(self.group)
            # padded all-gather of every rank's records and piece table
            loc = self._local()
            n = torch.tensor([len(loc), len(self.pieces)], dtype=torch.int64, device=dev)
            ns = torch.empty(2 * self.world, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(ns, n, group=self.group)
            ns = ns.view(self.world, 2).tolist()
            mb, mp = max(x[0] for x in ns), max(x[1] for x in ns)
            buf = torch.zeros(max(mb, 1), dtype=torch.uint8)
            if loc:
                buf[: len(loc)] = torch.frombuffer(bytearray(loc), dtype=torch.uint8)
            tab = torch.zeros(max(mp, 1) * 3, dtype=torch.int64)
            if self.pieces:
                tab[: 3 * len(self.pieces)] = torch.tensor([x for p in self.pieces for x in p], dtype=torch.int64)
            allb = torch.empty(self.world * max(mb, 1), dtype=torch.uint8, device=dev)
            allt = torch.empty(self.world * max(mp, 1) * 3, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(allb, buf.to(dev), group=self.group)
            dist.all_gather_into_tensor(allt, tab.to(dev), group=self.group)
            allb = allb.view(self.world, -1).cpu().numpy()
            allt = allt.view(self.world, -1, 3).cpu().tolist()
            parts = [([tuple(x) for x in allt[r][: ns[r][1]]], allb[r].tobytes()) for r in range(self.world)]
        for pieces, loc in parts:
            for so, lo, n in pieces:
                out[so: so + n] = loc[lo: lo + n]
        return bytes(out)


def split_frame(nbytes: int, element_type: int, flags: int, block_size: int, segment_count: int, buffer_size: int,
                rec_sizes: Sequence[int], crc: int):
    """(stream length, frame pieces, stream offset of every record) of a stream
    from its record sizes (stream.py:100-111, 271-284, 344-355)."""
    import struct

    from .stream import _WIDTH

    lay = stream_layout(nbytes, _WIDTH[element_type], bool(flags & 1), block_size, segment_count, buffer_size)
    offs = [0]
    for n in rec_sizes:
        offs.append(offs[-1] + int(n))
    frame = [(0, struct.pack("<4sBBBBQIII", b"LMC1", 1, flags, element_type, 0, nbytes, block_size, segment_count,
                             crc))]
    pos = 28
    rec_at = [0] * len(rec_sizes)
    for w in lay:
        tab = b"".join(struct.pack("<QQ", orig, offs[bb] - offs[ba]) for orig, ba, bb in w["segments"])
        frame.append((pos, tab))
        pos += len(tab)
        b0 = w["blk0"]
        for b in range(b0, b0 + w["nblocks"]):
            rec_at[b] = pos + offs[b] - offs[b0]
        pos += offs[b0 + w["nblocks"]] - offs[b0]
    return pos, frame, rec_at


def compress_split(tensor, *, group=None, element_type: int | None = None, prev=None, byte_group: bool = True,
                   block_size: int = 65536, segment_count: int = 1, buffer_size: int = 128 << 20,
                   codec=None, part_fn: Callable | None = None) -> SplitStream:
    """Compress ONE tensor with all ranks of ``group`` (each holds the whole
    tensor, e.g. replicated parameters): rank r compresses its block range;
    one all-gather of (record sizes, raw CRC) -- sizes only, the records stay
    where they were made -- gives every rank the stream's layout.  The result
    (a SplitStream) writes this rank's records at their final offsets; the
    assembled stream is byte-identical to a one-GPU lmc_compress.

    ``part_fn(blk_a, blk_b, crc_a, crc_b) -> (records: bytes, sizes: list,
    raw_crc: int)`` replaces the GPU part compression (tests drive the
    exchange logic on CPU with it)."""
    import torch
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
    dev = collective_device(group)
    if part_fn is None:
        codec = codec or __import__("paper_2505_09810_b200").stream.default_codec()
        rec, sizes_d, crc_d = codec.compress_part(tensor, ba, bb, ca, cb, element_type=et, prev=prev,
                                                  byte_group=byte_group, block_size=block_size,
                                                  segment_count=segment_count, buffer_size=buffer_size)
        mine = torch.cat([sizes_d.to(torch.int64), crc_d.to(torch.int64)]).to(dev)
        records = rec
    else:
        recs_b, sizes, raw = part_fn(ba, bb, ca, cb)
        mine = torch.tensor(list(sizes) + [raw], dtype=torch.int64, device=dev)
        records = recs_b
    # padded all-gather of (sizes, crc): every rank knows every block range
    width = max(r[1] - r[0] for r in ranges) + 1
    vec = torch.zeros(width, dtype=torch.int64, device=dev)
    vec[: mine.numel()] = mine
    if world > 1:
        rows = torch.empty(world * width, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(rows, vec, group=group)
        rows = rows.view(world, width).cpu().tolist()
    else:
        rows = [vec.cpu().tolist()]
    all_sizes, crc_parts = [], []
    for r, (a, b, c0, c1) in enumerate(ranges):
        all_sizes += rows[r][: b - a]
        crc_parts.append((rows[r][b - a] & 0xFFFFFFFF, c1 - c0))
    flags = (1 if byte_group else 0) | (2 if prev is not None else 0)
    crc = crc_combine(crc_parts) if nbytes else 0
    length, frame, rec_at = split_frame(nbytes, et, flags, block_size, segment_count, buffer_size, all_sizes, crc)
    # this rank's records: contiguous runs between segment tables
    pieces, lo, b = [], 0, ba
    bounds = sorted({w["blk0"] for w in lay} | {w["blk0"] + w["nblocks"] for w in lay})
    while b < bb:
        e = min([x for x in bounds if x > b] + [bb])
        n = sum(all_sizes[b:e])
        if n:
            pieces.append((rec_at[b], lo, n))
        lo += n
        b = e
    return SplitStream(rank, world, length, frame, pieces, records, group)


def assemble_stream(nbytes: int, element_type: int, flags: int, block_size: int, segment_count: int,
                    buffer_size: int, rec_sizes: Sequence[int], records: bytes,
                    crc_parts: Sequence[tuple[int, int]]) -> bytes:
    """The LMC1 stream from all records (in record order, back to back), their
    sizes and the (raw CRC, length) of consecutive payload byte ranges."""
    crc = crc_combine(crc_parts) if nbytes else 0
    length, frame, rec_at = split_frame(nbytes, element_type, flags, block_size, segment_count, buffer_size,
                                        rec_sizes, crc)
    out = bytearray(length)
    for off, b in frame:
        out[off: off + len(b)] = b
    pos = 0
    for i, n in enumerate(rec_sizes):
        out[rec_at[i]: rec_at[i] + n] = records[pos: pos + n]
        pos += n
    return bytes(out)


def _nbytes(t) -> int:
    if t is None:
        raise ValueError("tensor sizes are needed for unowned entries: pass nbytes=")
    if hasattr(t, "data") and isinstance(t.data, (bytes, bytearray, memoryview)):
        return len(t.data)        # TensorBuffer / DeltaBuffer (types.py)
    if hasattr(t, "numel"):
        return int(t.numel() * t.element_size())
    return int(np.asarray(t).nbytes)
