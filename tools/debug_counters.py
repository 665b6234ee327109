"""Build a -DLMCG_DEBUG variant of the library and print decode counters on cfg2 (GPU box)."""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_09810_b200 import _build, _lib
so = os.path.join(ROOT, "gpurun_out", "liblmc_b200_dbg.so")
if True:
    subprocess.check_call(["nvcc", *_build.NVCC_FLAGS, "-DLMCG_DEBUG", "-o", so, os.path.join(_build.SRC_DIR, "capi.cu")])
_lib.SO_PATH = so
L = _lib.load(so)
import torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
specs, ts = synth.make_checkpoint(cfg, seed=5)
codec = lmcb.Codec()
b = codec.compress(ts)
cnt = (ctypes.c_ulonglong * 32)()
L.lmcg_debug_counters(cnt, 1)
r = codec.decompress(b)
L.lmcg_debug_counters(cnt, 1)
names = ["m0 calls", "m0 syms", "m1 calls", "m1 syms", "m2 calls", "m2 syms", "m3 calls", "m3 syms", "fixup rounds", "-", "-", "-",
         "-", "-", "-", "-", "huff setup cyc", "staged recs", "pass0 cyc", "fixup cyc", "emit cyc", "chunks", "scan cyc",
         "lookback cyc", "huff rec cyc", "rle rec cyc", "stored rec cyc", "-", "huff recs", "rle recs", "stored recs"]
for i, n in enumerate(names):
    print(f"{n:14s} {cnt[i]}")
print("status", set(r.status))
