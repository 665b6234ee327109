import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth, _lib
specs, ts = synth.make_checkpoint("cfg2", seed=1)
codec = lmcb.Codec()
b = codec.compress(ts)
r = codec.decompress(b)
torch.cuda.synchronize()
L = codec.ctx.lib
off, ln = b.host_layout()
n = len(ts)
streams = [b.data[o:o+k] for o, k in zip(off, ln)]
ptrs = (ctypes.c_void_p * n)(*[v.data_ptr() for v in streams])
lens = (ctypes.c_uint64 * n)(*[v.numel() for v in streams])
hs = (_lib.lmcg_stream_hint * n)()
for i, h in enumerate(b.hints):
    hs[i].orig, hs[i].segments, hs[i].block, hs[i].windows = h
pos = 0; offs = []
for h in b.hints:
    offs.append(pos); pos += (h[0] + 15) & ~15
out = torch.empty(pos, dtype=torch.uint8, device="cuda")
hoff = (ctypes.c_uint64 * n)(*offs)
st = (ctypes.c_int32 * n)()
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = L.lmcg_decompress(codec.ctx.ptr, ptrs, lens, n, hs, out.data_ptr(), out.numel(), hoff, None)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rc2 = L.lmcg_decompress_result(codec.ctx.ptr, n, st, None, None, None, None)
    t3 = time.perf_counter()
    print(f"decompress call {1e3*(t1-t0):.3f} ms, gpu drain {1e3*(t2-t1):.3f} ms, result {1e3*(t3-t2):.3f} ms rc={rc},{rc2}")
codec.ctx.profile(True)
L.lmcg_decompress(codec.ctx.ptr, ptrs, lens, n, hs, out.data_ptr(), out.numel(), hoff, None)
print(codec.ctx.profile_report())
