"""Worker of tests/test_shard_nccl.py, launched with torch.distributed.run:
one rank per GPU under NCCL.  A small checkpoint is sharded across the ranks
(whole tensors, `shard.compress_sharded` with CUDA tensors -> the GPU codec),
the only exchange is the all-gather of stream lengths (device tensors), every
rank pwrites its streams into the shared packed file, and one tensor is also
split by block range (`shard.compress_split`: record sizes and CRCs
exchanged, records stay on their rank).  Rank 0 compares everything with the
oracle.  usage: _nccl_worker.py OUTDIR
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np   # noqa: E402
import torch         # noqa: E402
import torch.distributed as dist   # noqa: E402


def main():
    out_dir = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_09810_b200 import shard, synth
    from oracle import oracle as O

    # every rank generates the same seeded tensors (a rank only needs its own)
    gen = torch.Generator(device="cuda").manual_seed(7)
    shapes = [(1024, 1024), (768, 3072), (3072, 768), (50257 // 8, 768), (768,), (2048, 2048), (1 << 20,)]
    ts = [(torch.randn(s, generator=gen, device="cuda") * 0.02).to(torch.bfloat16) for s in shapes]
    res = shard.compress_sharded(ts)
    path = os.path.join(out_dir, "ckpt.lmc")
    if rank == 0:
        with open(path, "wb") as f:
            f.truncate(res.total_bytes)
    dist.barrier()
    fd = os.open(path, os.O_WRONLY)
    try:
        res.write_into(fd)
    finally:
        os.close(fd)
    # one tensor split by block range across the ranks
    big = ts[5]
    sp = shard.compress_split(big)
    spath = os.path.join(out_dir, "split.lmc")
    if rank == 0:
        with open(spath, "wb") as f:
            f.truncate(sp.length)
    dist.barrier()
    fd = os.open(spath, os.O_WRONLY)
    try:
        sp.write_into(fd)
    finally:
        os.close(fd)
    dist.barrier()
    if rank == 0:
        raw = [t.view(torch.uint8).reshape(-1).cpu().numpy().tobytes() for t in ts]
        want = [O.compress(r, 1, threads=4) for r in raw]
        packed = open(path, "rb").read()
        ok_packed = packed == b"".join(want)
        ok_lengths = res.lengths == [len(w) for w in want]
        ok_split = open(spath, "rb").read() == want[5]
        owners = sorted(set(res.owner))
        json.dump({"world": world, "packed": ok_packed, "lengths": ok_lengths, "split": ok_split, "owners": owners,
                   "backend": dist.get_backend()}, open(os.path.join(out_dir, "result.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
