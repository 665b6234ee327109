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
specs, ts = synth.make_checkpoint(cfg, seed=int(sys.argv[2]) if len(sys.argv) > 2 else 5)
prev = None
if len(sys.argv) > 3 and sys.argv[3] == "delta":
    prev, ts = ts, [synth.next_step(w, 5, i) for i, w in enumerate(ts)]
codec = lmcb.Codec()
b = codec.compress(ts, prev=prev)
cnt = (ctypes.c_ulonglong * 32)()
L.lmcg_debug_counters(cnt, 1)
r = codec.decompress(b)
L.lmcg_debug_counters(cnt, 1)
print("first decompress: fallback segs", cnt[11], "dense", cnt[12], "r>=R", cnt[13], "recfail", cnt[14], "verify", cnt[15])
r = codec.decompress(b)
L.lmcg_debug_counters(cnt, 1)
names = ["count calls", "count syms", "rec-bm calls", "rec-bm syms", "emit calls", "emit syms", "fix nosync", "fix syms", "fixup rounds", "nosync last", "nosync p0bad", "fallback segs",
         "dense", "r>=R", "rec fail", "verify fail", "huff setup cyc", "staged recs", "pass0 cyc", "fixup cyc", "emit cyc", "pair fail", "interleave+crc cyc",
         "crc table cyc", "huff rec cyc", "rle rec cyc", "stored rec cyc", "nosync e2bad", "huff recs", "rle recs", "stored recs"]
for i, n in enumerate(names):
    print(f"{n:14s} {cnt[i]}")
print("status", set(r.status))
ev = (ctypes.c_ulonglong * 4096)()
L.lmcg_debug_events(ev)
for k in range(min(12, int(cnt[10]) if cnt[10] else 512)):
    e = ev[8 * k: 8 * k + 8]
    if e[5] == 0: break
    print("ev cta", e[0], "c", e[1], "p0", e[2], "pe", e[3], "lim", e[4], "bits", e[5], "min/max", e[6] >> 32, e[6] & 0xFFFFFFFF, "p0cnt/cnt2", e[7] >> 32, e[7] & 0xFFFFFFFF)
