"""Per-kernel times of compress + decompress on a synthetic config (no correctness gate; experiments)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
specs, ts = synth.make_checkpoint(cfg, seed=1000, device="cuda")
prev = None
if len(sys.argv) > 2 and sys.argv[2] == "delta":   # step t+1 against step t (fused XOR)
    prev, ts = ts, [synth.next_step(w, 1000, i) for i, w in enumerate(ts)]
codec = lmcb.Codec(0)
for _ in range(2):
    b = codec.compress(ts, prev=prev); r = codec.decompress(b)
codec.ctx.profile(True)
n = 3
for _ in range(n):
    b = codec.compress(ts, prev=prev); r = codec.decompress(b)
prof = codec.ctx.profile_report()
codec.ctx.profile(False)
print({k: round(v[1] / n, 4) for k, v in sorted(prof.items()) if v[1] / n > 0.005}, "status", set(r.status))
