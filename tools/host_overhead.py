import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
specs, ts = synth.make_checkpoint("cfg2", seed=1)
codec = lmcb.Codec()
for _ in range(3):
    b = codec.compress(ts); r = codec.decompress(b)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    b = codec.compress(ts)
torch.cuda.synchronize()
t1 = time.perf_counter()
for _ in range(10):
    r = codec.decompress(b)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"compress wall {(t1-t0)/10*1e3:.3f} ms  decompress wall {(t2-t1)/10*1e3:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    b = codec.compress(ts)
    r = codec.decompress(b)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
