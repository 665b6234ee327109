import ctypes, os, subprocess, sys
sys.path.insert(0, os.getcwd())
from paper_2505_09810_b200 import _build, _lib
so = os.path.join(os.getcwd(), "gpurun_out", "liblmc_b200_dbg.so")
subprocess.check_call(["nvcc", *_build.NVCC_FLAGS, "-DLMCG_DEBUG", "-o", so, os.path.join(_build.SRC_DIR, "capi.cu")])
_lib.SO_PATH = so
L = _lib.load(so)
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
if cfg == "cfg4":
    specs, prev = synth.make_checkpoint("cfg4", seed=5, limit=14)
    nxt = [synth.next_step(w, 5, i) for i, w in enumerate(prev)]
else:
    specs, nxt = synth.make_checkpoint(cfg, seed=3)
    prev = None
codec = lmcb.Codec()
b = codec.compress(nxt, prev=prev)
info = codec.block_info()
import collections
print("modes", collections.Counter(info["modes"].tolist()) if hasattr(info["modes"], "tolist") else info.keys())
cnt = (ctypes.c_ulonglong * 32)()
L.lmcg_debug_counters(cnt, 1)
r = codec.decompress(b)
L.lmcg_debug_counters(cnt, 1)
print("resolved", cnt[9], "unresolved", cnt[10], "decode fail", cnt[16], "fallback segs", cnt[11], "lane-dense", cnt[12], "r>=R", cnt[13], "recfail", cnt[14], "verify", cnt[15], "status", set(r.status))
off, ln = b.host_layout()
print("streams", len(ln), "sizes", ln[:6])
