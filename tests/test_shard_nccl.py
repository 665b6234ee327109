"""One rank per GPU under NCCL (torch.distributed.run): a checkpoint sharded
by whole tensors and one tensor split by block range, GPU codec on every
rank, only lengths / record sizes / CRCs exchanged (device tensors), every
rank writing its streams at their final offsets -- the packed file and the
split stream must equal the oracle's, byte for byte (the
reference's segment-level parallelism: parallel.py:86-103, stream.py:271-284).

Runs with two ranks when the box has two GPUs; on a one-GPU box the same
program runs as a one-rank NCCL job, which still drives every collective
with device tensors (a CPU tensor in an NCCL collective fails at world 1
as well)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world: int, tmp_path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_nccl_worker.py"), str(tmp_path)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    return json.load(open(os.path.join(tmp_path, "result.json")))


@pytest.mark.gpu
def test_nccl_sharded_checkpoint_and_split_tensor(tmp_path):
    import torch

    world = min(2, torch.cuda.device_count())
    assert world >= 1
    r = _run(world, tmp_path)
    assert r["backend"] == "nccl" and r["world"] == world
    assert r["packed"], "packed checkpoint differs from the oracle's streams"
    assert r["lengths"], "gathered stream lengths differ from the oracle's"
    assert r["split"], "the block-range split stream differs from the one-call stream"
    assert r["owners"] == list(range(world))     # every rank compressed something
