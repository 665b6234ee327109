"""GPU box: replay cfg5 compress+decompress plans and report decode failures per stream."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
graph = (sys.argv[2] if len(sys.argv) > 2 else "1") == "1"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
specs, ts = synth.make_checkpoint(cfg, seed=5)
codec = lmcb.Codec()
cp = codec.compress_plan(ts, graph=graph)
dp = cp.decompress_plan(graph=graph)
bad_total = 0
for it in range(reps):
    b = cp.run()
    r = dp.run(b)
    st = r.status
    bad = [i for i, s in enumerate(st) if s]
    mism = [i for i, t in enumerate(ts) if not torch.equal(r.payload(i), t.view(torch.uint8).reshape(-1))]
    if bad or mism:
        bad_total += 1
        print("iter", it, "bad status", [(i, st[i], specs[i].name, tuple(ts[i].shape)) for i in bad[:8]], "mismatch", mism[:8], flush=True)
        for i in (bad or mism)[:2]:
            t = ts[i].view(torch.uint8).reshape(-1)
            p = r.payload(i)
            d = (p != t).nonzero()
            if d.numel():
                print("  stream", i, "first diff byte", int(d[0]), "ndiff", d.numel(), "len", t.numel(), flush=True)
print("iterations with failures:", bad_total, "of", reps)
# interleave eager runs (the bench's profiling pass) with plan replays
for it in range(6):
    pb = codec.compress(ts)
    pb.host_layout()
    rr = codec.decompress(pb)
    if any(rr.status):
        print("eager iter", it, "bad", [(i, s) for i, s in enumerate(rr.status) if s][:8], flush=True)
    b = cp.run()
    r = dp.run(b)
    if any(r.status):
        print("plan-after-eager iter", it, "bad", [(i, s, specs[i].name) for i, s in enumerate(r.status) if s][:8], flush=True)
print("done")
