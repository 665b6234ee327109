import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
specs, ts = synth.make_checkpoint("cfg2", seed=1000, device="cuda")
codec = lmcb.Codec(0)
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
cp = codec.compress_plan(ts, graph=True); dp = cp.decompress_plan(graph=True)
def one():
    cp.run(); dp.run()
print("single", timeit(one))
for K in (2, 3, 4):
    # K groups balanced by bytes (largest first)
    order = sorted(range(len(ts)), key=lambda i: -ts[i].numel())
    groups = [[] for _ in range(K)]; load = [0]*K
    for i in order:
        g = min(range(K), key=lambda q: load[q]); groups[g].append(i); load[g] += ts[i].numel()
    plans = []
    for g in groups:
        c = codec.compress_plan([ts[i] for i in g], graph=True)
        plans.append((c, c.decompress_plan(graph=True)))
    streams = [torch.cuda.Stream() for _ in range(K)]
    main = torch.cuda.current_stream()
    def multi():
        for (c, d), st in zip(plans, streams):
            st.wait_stream(main)
            with torch.cuda.stream(st):
                c.run(); d.run()
        for st in streams: main.wait_stream(st)
    print("K", K, timeit(multi))
