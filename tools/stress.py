"""GPU box: replay compress/decompress plans (as bench.measure does) until a
decode status is bad; then classify the failing stream (compress or decode
side) against the oracle and eager decodes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if os.environ.get("STRESS_DEFS"):   # an experiment build of the library (extra -D flags), kept under gpurun_out/
    import subprocess
    from paper_2505_09810_b200 import _build, _lib as _l0
    so = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "liblmc_b200_exp.so")
    subprocess.check_call(["nvcc", *_build.NVCC_FLAGS, *os.environ["STRESS_DEFS"].split(), "-o", so, os.path.join(_build.SRC_DIR, "capi.cu")])
    _l0.SO_PATH = so
    _l0.load(so)
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
from paper_2505_09810_b200 import _lib
L = _lib.load()
L.lmcg_fallback_segments(1)
if os.environ.get("STRESS_NOFUSE"):
    codec.ctx.set_decode_fusion(False)
cp = codec.compress_plan(ts, prev=prev, graph=True)
dp = cp.decompress_plan(graph=True)
t0 = time.time()
nfail = 0
for it in range(reps):
    if it % 10 == 5 and not os.environ.get("STRESS_NOEAGER"):   # the bench's eager profiling pass
        pb = codec.compress(ts, prev=prev); pb.host_layout(); codec.decompress(pb)
    b = cp.run()
    r = dp.run(b)
    st = r.status
    bad = [i for i, s in enumerate(st) if s]
    fb = L.lmcg_fallback_segments(1) if os.environ.get("STRESS_SYNC") else 0
    if fb:
        print(f"iter {it}: {fb} segments took the serial fallback; bad streams {len(bad)}", flush=True)
        if "LMCG_DEBUG" in os.environ.get("STRESS_DEFS", ""):
            import ctypes
            ev = (ctypes.c_ulonglong * 4096)()
            L.lmcg_debug_events(ev)
            for k in range(512):
                e = ev[8 * k: 8 * k + 8]
                if e[3] == 0: break
                print(f"  ev cta {e[0]} tid {e[1]} first word {e[2]} (byte {4 * e[2]}) words {e[3]} got {e[4]:08x} want {e[5]:08x} pair {e[6]} clk {e[7]}", flush=True)
    if not bad:
        continue
    nfail += 1
    print(f"iter {it}: {len(bad)} bad streams", [(i, st[i], specs[i].name) for i in bad[:6]], flush=True)
    for i in bad:   # where does the payload differ from the input?
        want = (ts[i].view(torch.uint8) ^ prev[i].view(torch.uint8) if delta else ts[i].view(torch.uint8)).reshape(-1)
        got = r.payload(i)
        if got.numel() != want.numel():
            print(f"  stream {i}: payload length {got.numel()} != {want.numel()}", flush=True)
            continue
        d = torch.nonzero(got != want).reshape(-1)
        if d.numel() == 0:
            print(f"  stream {i}: payload bytes all equal (CRC-only failure)", flush=True)
        else:
            lo, hi = int(d[0]), int(d[-1])
            odd = int((d % 2 == 1).sum())
            print(f"  stream {i}: {d.numel()} bytes differ, first {lo} (pair {lo // 131072}, +{lo % 131072}) last {hi} (pair {hi // 131072}, +{hi % 131072}); odd-offset (high-plane) bytes {odd}", flush=True)
            k = lo
            print("    got ", got[k:k + 32].cpu().tolist(), flush=True)
            print("    want", want[k:k + 32].cpu().tolist(), flush=True)
    if os.environ.get("STRESS_SHORT"):
        if nfail >= 2: break
        continue
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
