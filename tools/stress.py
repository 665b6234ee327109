"""GPU box: replay compress/decompress plans (as bench.measure does) until a
decode status is bad; then classify the failing stream (compress or decode
side) against the oracle and eager decodes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
from oracle import oracle as O
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
delta = len(sys.argv) > 3 and sys.argv[3] == "delta"
specs, ts = synth.make_checkpoint(cfg, seed=5)
prev = None
if delta:
    prev, ts = ts, [synth.next_step(w, 5, i) for i, w in enumerate(ts)]
codec = lmcb.Codec()
cp = codec.compress_plan(ts, prev=prev, graph=True)
dp = cp.decompress_plan(graph=True)
t0 = time.time()
nfail = 0
for it in range(reps):
    if it % 10 == 5:   # the bench's eager profiling pass
        pb = codec.compress(ts, prev=prev); pb.host_layout(); codec.decompress(pb)
    b = cp.run()
    r = dp.run(b)
    st = r.status
    bad = [i for i, s in enumerate(st) if s]
    if not bad:
        continue
    nfail += 1
    print(f"iter {it}: {len(bad)} bad streams", [(i, st[i], specs[i].name) for i in bad[:6]], flush=True)
    streams = b.to_bytes()
    for i in bad[:3]:
        raw = (ts[i].view(torch.uint8) ^ prev[i].view(torch.uint8) if delta else ts[i].view(torch.uint8)).reshape(-1).cpu().numpy().tobytes()
        ref = O.compress(raw, 1, delta=delta, threads=16)
        same = streams[i] == ref
        print(f"  stream {i}: len {len(streams[i])} oracle len {len(ref)} identical={same}", flush=True)
        if not same:
            d = next((k for k in range(min(len(ref), len(streams[i]))) if ref[k] != streams[i][k]), None)
            print("   first differing byte", d, flush=True)
        try:
            O.decompress(streams[i]); oc = 0
        except O.OracleError as e:
            oc = e.code
        rr = codec.decompress([b.stream(i)])
        print(f"   oracle decode code {oc}; eager GPU decode status {rr.status}", flush=True)
    if nfail >= 3:
        break
print("fails", nfail, "of", it + 1, "in", round(time.time() - t0, 1), "s")
