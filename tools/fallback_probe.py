import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
specs, ts = synth.make_checkpoint("cfg2", seed=1)
codec = lmcb.Codec()
codec.ctx.profile(True)
seq = sys.argv[1] if len(sys.argv) > 1 else "cdddcdcd"
b = None
for op in seq:
    if op == "c":
        b = codec.compress(ts)
    else:
        r = codec.decompress(b)
    rep = codec.ctx.profile_report()
    print(op, {k: round(v[1], 3) for k, v in rep.items() if k in ("k_scandec", "k_fallback", "k_encode")})
