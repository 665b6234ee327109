"""compute-sanitizer target: compress + decompress (eager, fused and unfused
decode, plain and delta, aligned and 16-byte-offset views) of a small
checkpoint whose streams end exactly at the end of their device buffer.
usage: compute-sanitizer --tool memcheck python tools/san_roundtrip.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb

g = torch.Generator(device="cuda").manual_seed(3)
codec = lmcb.Codec()
for fuse in (True, False):
    codec.ctx.set_decode_fusion(fuse, 1)      # fused decode from one record slot on
    for off in (0, 16):
        n = 1 << 19
        base = torch.zeros(2 * n + 64, dtype=torch.uint8, device="cuda")
        w = (torch.randn(n, generator=g, device="cuda") * 0.02).to(torch.bfloat16)
        base[off: off + 2 * n] = w.view(torch.uint8)
        cur = base[off: off + 2 * n].view(torch.bfloat16)
        prev = (cur.float() * (1 + 1e-3 * torch.randn(n, generator=g, device="cuda"))).to(torch.bfloat16)
        ts = [cur, (torch.randn(3 * 16384 + 8, generator=g, device="cuda") * 0.02).to(torch.float16),
              torch.zeros(70000, dtype=torch.bfloat16, device="cuda")]
        for pv in (None, [prev, None, None]):
            b = codec.compress(ts if pv is None else ts[:1], prev=None if pv is None else pv[:1])
            # decode from exactly-sized stream tensors (every stream ends at its allocation's end)
            streams = [torch.empty(len(s), dtype=torch.uint8, device="cuda").copy_(torch.frombuffer(bytearray(s), dtype=torch.uint8)) for s in b.to_bytes()]
            r = codec.decompress(streams)
            assert set(r.status) == {0}, r.status
            want = cur.view(torch.uint8) if pv is None else cur.view(torch.uint8) ^ prev.view(torch.uint8)
            assert torch.equal(r.payload(0), want)
torch.cuda.synchronize()
print("ok")
