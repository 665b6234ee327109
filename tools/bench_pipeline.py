"""Checkpoint save with compression overlapped with D2H and file writes
(SURVEY §8(f) row 3), one JSON line.

For one config's checkpoint (resident on the GPU; delta configs compress
step t+1 against step t) it times, wall clock, files on local disk:

* serial: one batched compress, then D2H of all streams, then the file
  writes (what a caller without the pipeline does; the reference's
  chain.add_step is compress-write per stream, chain.py:185-196);
* pipelined: pipeline.StreamWriter (compress group g | D2H group g-1 |
  write group g-2) at a few group sizes;
* the stages alone: GPU compress (CUDA events), D2H of the streams, and the
  file writes from host memory -- the pipelined time is bounded below by the
  slowest stage.

usage: python tools/bench_pipeline.py [--config cfg2] [--dir /tmp/pipebench] [--reps 3]
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
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--dir", default="/tmp/pipebench")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--groups", default="64,256,1024")
    args = ap.parse_args()

    import torch

    import paper_2505_09810_b200 as lmcb
    from paper_2505_09810_b200 import synth
    from paper_2505_09810_b200.pipeline import StreamWriter, items_from_tensors

    torch.cuda.set_device(0)
    specs, ts = synth.make_checkpoint(args.config, seed=1000, device="cuda")
    prev = None
    if args.config in ("cfg4",):
        prev = ts
        ts = [synth.next_step(w, 1000, i) for i, w in enumerate(ts)]
    nbytes = sum(t.numel() * t.element_size() for t in ts)
    codec = lmcb.default_codec()
    names = [s.name.replace("/", "_") for s in specs]
    d = args.dir
    shutil.rmtree(d, ignore_errors=True)
    os.makedirs(d)
    paths = [os.path.join(d, n + ".lmc") for n in names]

    def write_all(streams):
        for p, s in zip(paths, streams):
            with open(p, "wb") as f:
                f.write(s)

    def serial():
        b = codec.compress(ts, prev=prev)
        write_all(b.to_bytes())

    def best(fn):
        fn()   # warm-up (allocations, page cache of the output files)
        torch.cuda.synchronize()
        ts_ = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts_.append(time.perf_counter() - t0)
        return min(ts_)

    res = {"config": args.config, "bytes": nbytes, "tensors": len(ts), "dir": d}
    # stages alone
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b = codec.compress(ts, prev=prev)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        b = codec.compress(ts, prev=prev)
    e1.record()
    torch.cuda.synchronize()
    res["gpu_compress_ms"] = round(e0.elapsed_time(e1) / 3, 3)
    total = b.total_bytes()
    res["stream_bytes"] = total
    pin = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    t_d2h = best(lambda: pin.copy_(b.data[:total], non_blocking=True))
    res["d2h_ms"] = round(1e3 * t_d2h, 2)
    streams = b.to_bytes()
    res["write_ms"] = round(1e3 * best(lambda: write_all(streams)), 2)
    # serial and pipelined
    t_ser = best(serial)
    res["serial_ms"] = round(1e3 * t_ser, 2)
    res["serial_gib_s"] = round(nbytes / GIB / t_ser, 3)
    items = items_from_tensors(ts, prev)

    def sink(i, view):
        with open(paths[i], "wb") as f:
            f.write(view)

    w = StreamWriter(codec, group_bytes=256 << 20)
    res["pipelined_256MiB_nowrite_ms"] = round(1e3 * best(lambda: w.run(items, lambda i, v: None)), 2)
    for g in [int(x) for x in args.groups.split(",")]:
        for nw in (1, 4):
            w = StreamWriter(codec, group_bytes=g << 20, writers=nw)
            t = best(lambda: w.run(items, sink))
            res[f"pipelined_{g}MiB_w{nw}_ms"] = round(1e3 * t, 2)
            res[f"pipelined_{g}MiB_w{nw}_gib_s"] = round(nbytes / GIB / t, 3)
    # the files are the one-batch streams
    for p, s in zip(paths, streams):
        with open(p, "rb") as f:
            assert f.read() == s, p
    shutil.rmtree(d, ignore_errors=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
