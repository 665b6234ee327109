"""Checkpoint-chain throughput on one GPU, one JSON line.

Workload: cfg4 (GPT-style 1.3B, 292 bf16 tensors, 2.45 GiB per step) and its
next step under the survey's delta model.  Measured with CUDA events on the
device, inputs resident in HBM:

* add: ``Codec.compress(step1, prev=step0)`` -- the XOR fused into the
  compress loads -- plus the device copy that makes step 1 the resident step
  (what DeviceChain.add_step does on the device);
* apply: ``Codec.decompress(delta, prev=resident, out=resident)`` -- decode
  fused with xor_apply, in place (DeviceChain.restore_step's per-step work);

and end to end (wall clock, files on local disk under /tmp):
``DeviceChain.add_step`` of both steps and ``restore_step(1)`` from a fresh
object.  The CPU column is the C oracle port on a bounded sample: decode the
delta and XOR onto the previous step (chain.py:293-300's per-step work).

usage: python tools/bench_chain.py [--steps K] [--warmup W] [--dir /tmp/chainbench]
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

GIB = float(1 << 30)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dir", default="/tmp/chainbench")
    ap.add_argument("--config", default="cfg4")
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2505_09810_b200 as lmcb
    from paper_2505_09810_b200 import synth

    torch.cuda.set_device(0)
    specs, s0 = synth.make_checkpoint(args.config, seed=1000, device="cuda")
    s1 = [synth.next_step(w, 1000, i) for i, w in enumerate(s0)]
    names = [s.name for s in specs]
    nbytes = sum(t.numel() * 2 for t in s0)
    codec = lmcb.Codec(0)

    # resident buffer laid out like DeviceChain's
    offs, pos = [], 0
    for t in s0:
        offs.append(pos)
        pos += (t.numel() * 2 + 15) & ~15
    res = torch.empty(pos, dtype=torch.uint8, device="cuda")
    views = [res[o: o + t.numel() * 2] for o, t in zip(offs, s0)]
    flat1 = [t.view(torch.uint8).reshape(-1) for t in s1]
    flat0 = [t.view(torch.uint8).reshape(-1) for t in s0]

    def load_step0():
        for v, x in zip(views, flat0):
            v.copy_(x)

    # correctness first: add (delta vs resident step 0), then apply in place
    load_step0()
    batch = codec.compress(s1, prev=views)
    stream_bytes = batch.total_bytes()
    r = codec.decompress(batch, out=res, out_offsets=offs, prev=views)
    r.raise_for_status()
    for v, x in zip(views, flat1):
        assert torch.equal(v, x), "apply mismatch"

    st = torch.cuda.current_stream()
    delta = batch
    add_ms, apply_ms = [], []
    for k in range(args.warmup + args.steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        load_step0()
        torch.cuda.synchronize()
        e[0].record(st)
        batch = codec.compress(s1, prev=views)
        for v, x in zip(views, flat1):     # step 1 becomes the resident step
            v.copy_(x)
        e[1].record(st)
        load_step0()
        e[2].record(st)
        r = codec.decompress(delta, out=res, out_offsets=offs, prev=views)
        e[3].record(st)
        torch.cuda.synchronize()
        if k >= args.warmup:
            add_ms.append(e[0].elapsed_time(e[1]))
            apply_ms.append(e[2].elapsed_time(e[3]))
    r.raise_for_status()
    add = float(np.median(add_ms))
    app = float(np.median(apply_ms))

    # end to end through DeviceChain (files under --dir)
    shutil.rmtree(args.dir, ignore_errors=True)
    ch = lmcb.DeviceChain(args.dir)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ch.add_step(dict(zip(names, s0)))
    t1 = time.perf_counter()
    ch.add_step(dict(zip(names, s1)))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    fresh = lmcb.DeviceChain(args.dir)
    got = fresh.restore_step(1)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    for n, x in zip(names, flat1):
        assert torch.equal(got[n], x), n
    disk = sum(os.path.getsize(os.path.join(args.dir, f)) for f in os.listdir(args.dir))
    shutil.rmtree(args.dir, ignore_errors=True)

    # CPU: oracle port on a bounded sample (decode the delta, XOR onto step 0)
    from oracle import oracle as O

    cores = os.cpu_count() or 1
    sample, nb = [], 0
    for i in range(2, len(s0)):
        d = (flat1[i] ^ flat0[i]).cpu().numpy().tobytes()
        sample.append((O.compress(d, 1, delta=True, threads=cores), flat0[i].cpu().numpy()))
        nb += len(d)
        if nb >= 64 << 20:
            break
    tc0, reps = time.perf_counter(), 0
    while True:
        for s, p in sample:
            out = np.frombuffer(O.decompress(s, threads=cores)[0], np.uint8) ^ p
        reps += 1
        if time.perf_counter() - tc0 > 8.0:
            break
    cpu = nb * reps / (time.perf_counter() - tc0) / GIB
    line = {
        "metric": "chain step throughput (uncompressed GiB/s per step)",
        "config": {"workload": f"{args.config}: GPT-style 1.3B, {len(s0)} bf16 tensors, step t -> t+1 delta model "
                               "(SURVEY §8(d)), default options"},
        "step_bytes": nbytes, "delta_stream_bytes": stream_bytes, "ratio": round(stream_bytes / nbytes, 5),
        "device": {"add_ms": round(add, 3), "add_gib_s": round(nbytes / add * 1e3 / GIB, 2),
                   "apply_ms": round(app, 3), "apply_gib_s": round(nbytes / app * 1e3 / GIB, 2),
                   "steps": args.steps, "warmup": args.warmup,
                   "add": "compress(step1, prev=resident) + D2D refresh of the resident step",
                   "apply": "decompress(delta, prev=resident, out=resident): decode + xor_apply in place"},
        "e2e_wall_s": {"add_step0": round(t1 - t0, 3), "add_step1": round(t2 - t1, 3),
                       "restore_step1_fresh": round(t3 - t2, 3), "chain_bytes_on_disk": disk},
        "cpu_baseline": {"value": round(cpu, 4), "unit": "GiB/s", "cores": cores, "kind": "port",
                         "sample": f"{len(sample)} delta streams ({nb / 2**20:.1f} MiB): oracle decode + numpy XOR"},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
