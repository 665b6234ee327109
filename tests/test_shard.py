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
