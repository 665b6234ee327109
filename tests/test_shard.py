"""Multi-rank sharding of a checkpoint (paper_2505_09810_b200/shard.py) on CPU.

world_size-2 ``gloo`` process groups on 127.0.0.1 exercise the host logic of
the multi-GPU path: the owner table, the all-gather of compressed sizes, the
manifest and the per-rank pwrite of streams into one packed file.  Per-rank
compression is injected (the C oracle) because there is no GPU here; the GPU
codec is the default ``compress_fn`` and is covered by tests/test_gpu_parity.py.
The packed file must be byte-identical to the streams a single process writes.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2505_09810_b200 import shard

BF16 = 1


def _tensors(seed=3):
    rng = np.random.default_rng(seed)
    sizes = [70000, 4096, 131072, 2 * 65536 + 10, 8192, 2, 200000, 0, 65536]
    out = []
    for n in sizes:
        v = (rng.normal(0, 0.02, n).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        out.append(v.tobytes())
    return out


def _oracle_fn(bufs):
    return [O.compress(b, BF16, block_size=65536, threads=1) for b in bufs]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, path, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ts = _tensors()
        # unowned tensors are not needed on a rank: pass sizes instead
        nbytes = [len(t) for t in ts]
        owner = shard.assign_tensors(nbytes, world)
        mine = [t if owner[i] == rank else None for i, t in enumerate(ts)]
        res = shard.compress_sharded(mine, nbytes=nbytes, compress_fn=_oracle_fn)
        fd = os.open(path, os.O_RDWR)
        try:
            res.write_into(fd)
        finally:
            os.close(fd)
        dist.barrier()
        with open(path, "rb") as f:
            packed = f.read()
        dec = shard.decompress_sharded(packed, res.lengths, res.owner, rank=rank,
                                       decompress_fn=lambda ss: [O.decompress(s)[0] for s in ss])
        ok = all(dec[i] == ts[i] for i in dec)
        q.put((rank, res.owned, res.lengths, res.offsets, ok))
    finally:
        dist.destroy_process_group()


def test_assign_is_balanced_and_deterministic():
    sizes = [5, 9, 9, 1, 7, 3, 3, 100]
    a = shard.assign_tensors(sizes, 3)
    assert a == shard.assign_tensors(sizes, 3)
    assert a[7] == 0 and a[1] == 1 and a[2] == 2          # largest first, ties by index
    loads = [sum(s for s, r in zip(sizes, a) if r == q) for q in range(3)]
    assert max(loads) == 100
    assert shard.assign_tensors(sizes, 1) == [0] * len(sizes)
    with pytest.raises(ValueError):
        shard.assign_tensors(sizes, 0)


def test_manifest_offsets():
    assert shard.manifest_offsets([3, 0, 5]) == [0, 3, 3]
    assert shard.manifest_offsets([], 7) == []


def test_single_process_matches_serial():
    ts = _tensors()
    res = shard.compress_sharded(ts, compress_fn=_oracle_fn)
    assert res.world == 1 and res.owned == list(range(len(ts)))
    streams = _oracle_fn(ts)
    assert res.lengths == [len(s) for s in streams]
    assert res.total_bytes == sum(len(s) for s in streams)


def test_gloo_world2_packed_file_identical():
    ts = _tensors()
    streams = _oracle_fn(ts)
    want = b"".join(streams)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ckpt.lmc")
        with open(path, "wb") as f:
            f.truncate(len(want))
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, path, q)) for r in range(2)]
        for p in procs:
            p.start()
        got = [q.get(timeout=120) for _ in procs]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        with open(path, "rb") as f:
            packed = f.read()
    assert packed == want
    got.sort()
    owned = sorted(got[0][1] + got[1][1])
    assert owned == list(range(len(ts)))                 # every tensor exactly once
    assert got[0][1] and got[1][1]                        # both ranks did work
    for _, _, lengths, offsets, ok in got:
        assert lengths == [len(s) for s in streams]
        assert offsets == shard.manifest_offsets(lengths)
        assert ok


@pytest.mark.gpu
def test_single_rank_gpu_codec_matches_oracle():
    from paper_2505_09810_b200.types import ElementType, TensorBuffer

    ts = _tensors()
    res = shard.compress_sharded([TensorBuffer(t, ElementType.BF16) for t in ts])
    streams = _oracle_fn(ts)
    assert [res.streams[i] for i in range(len(ts))] == streams
    packed = b"".join(streams)
    dec = shard.decompress_sharded(packed, res.lengths, res.owner, rank=0)
    assert all(dec[i].data == ts[i] for i in range(len(ts)))


# ------------------------------------------------ one tensor, several ranks
def _records(stream):
    """(sizes, concatenated records) of an LMC1 stream, in record order."""
    import struct
    hdr = struct.unpack_from("<4sBBBBQIII", stream, 0)
    orig, B, S = hdr[5], hdr[6], hdr[7]
    pos, sizes, recs = 28, [], []
    left = orig
    while left > 0:
        tab = [struct.unpack_from("<QQ", stream, pos + 16 * i) for i in range(S)]
        pos += 16 * S
        for o, c in tab:
            end = pos + c
            while pos < end:
                mode, L = stream[pos], struct.unpack_from("<I", stream, pos + 1)[0]
                n = 5 + (1 if mode == 1 else L if mode == 2 else 132 + (struct.unpack_from("<I", stream, pos + 133)[0] + 7) // 8)
                sizes.append(n)
                recs.append(stream[pos:pos + n])
                pos += n
            left -= o
    return sizes, b"".join(recs)


def _raw_crc(b):
    import zlib
    return zlib.crc32(b) ^ 0xFFFFFFFF ^ shard.crc_shift(0xFFFFFFFF, len(b))


def _oracle_part_fn(data, **opts):
    full = O.compress(data, BF16, threads=1, **opts)
    sizes, recs = _records(full)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    def part(ba, bb, ca, cb):
        return recs[offs[ba]:offs[bb]], sizes[ba:bb], _raw_crc(data[ca:cb])
    return full, part


def test_split_single_process_matches_oracle():
    for opts in ({"block_size": 4096, "segment_count": 3, "buffer_size": 40000}, {"block_size": 65536}):
        data = _tensors()[6]
        full, part = _oracle_part_fn(data, **opts)
        got = shard.compress_split(data, element_type=BF16, part_fn=part, **opts)
        assert got.length == len(full)
        assert got.to_bytes() == full


def _split_worker(rank, world, port, q, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data = _tensors()[6]
        opts = {"block_size": 4096, "segment_count": 3, "buffer_size": 40000}
        full, part = _oracle_part_fn(data, **opts)
        got = shard.compress_split(data, element_type=BF16, part_fn=part, **opts)
        # each rank writes only its own records (rank 0 also the frame) into
        # the shared file; records never cross ranks on this path
        fd = os.open(path, os.O_RDWR)
        try:
            got.write_into(fd)
        finally:
            os.close(fd)
        dist.barrier()
        with open(path, "rb") as f:
            on_disk = f.read()
        q.put((rank, on_disk == full and got.to_bytes() == full and got.length == len(full)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_split_one_tensor():
    data = _tensors()[6]
    full, _ = _oracle_part_fn(data, block_size=4096, segment_count=3, buffer_size=40000)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "split.lmc")
        with open(path, "wb") as f:
            f.truncate(len(full))
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q, path)) for r in range(2)]
        for p in procs:
            p.start()
        got = sorted(q.get(timeout=120) for _ in procs)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    assert got == [(0, True), (1, True)]


def test_pwrite_all_loops_until_written(tmp_path, monkeypatch):
    # os.pwrite may write fewer bytes than asked (Linux caps one call near 2 GiB)
    real = os.pwrite
    calls = []

    def short(fd, data, off):
        calls.append(off)
        return real(fd, bytes(data)[:3], off)

    monkeypatch.setattr(shard.os, "pwrite", short)
    p = tmp_path / "f"
    p.write_bytes(b"\0" * 20)
    fd = os.open(p, os.O_RDWR)
    try:
        shard._pwrite_all(fd, b"abcdefghij", 5)
    finally:
        os.close(fd)
    assert p.read_bytes() == b"\0" * 5 + b"abcdefghij" + b"\0" * 5
    assert calls == [5, 8, 11, 14]


def test_collective_device_defaults():
    import torch
    assert shard.collective_device() == torch.device("cpu")
    assert shard.collective_device(device="cpu") == torch.device("cpu")


@pytest.mark.gpu
def test_gpu_parts_assemble_to_the_one_call_stream():
    import torch
    from paper_2505_09810_b200 import synth
    import paper_2505_09810_b200 as lmcb

    codec = lmcb.Codec()
    t = synth.make_tensor(synth.TensorSpec("w", (4096, 4096), "weight"), 7, 0)
    p = synth.make_tensor(synth.TensorSpec("w", (4096, 4096), "weight"), 8, 0)
    for opts, prev in (({}, None), ({"block_size": 16384, "segment_count": 4, "buffer_size": 12 << 20}, None),
                       ({}, p)):
        b = codec.compress([t], prev=None if prev is None else [prev], **opts)
        want = b.to_bytes()[0]
        for world in (2, 3, 5):
            lay = shard.stream_layout(t.numel() * 2, 2, True, opts.get("block_size", 65536),
                                      opts.get("segment_count", 1), opts.get("buffer_size", 128 << 20))
            nblk = sum(w["nblocks"] for w in lay)
            sizes, recs, crcs = [], [], []
            for ba, bb, ca, cb in shard.split_ranges(nblk, t.numel() * 2, world):
                r, s, c = codec.compress_part(t, ba, bb, ca, cb, prev=prev, **opts)
                s = [int(x) for x in s.tolist()]
                sizes += s
                recs.append(r[:sum(s)].cpu().numpy().tobytes())
                crcs.append((int(c.item()) & 0xFFFFFFFF, cb - ca))
            got = shard.assemble_stream(t.numel() * 2, 1, 1 | (2 if prev is not None else 0),
                                        opts.get("block_size", 65536), opts.get("segment_count", 1),
                                        opts.get("buffer_size", 128 << 20), sizes, b"".join(recs), crcs)
            assert got == want, (opts.keys(), world)
