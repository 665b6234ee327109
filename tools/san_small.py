import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_09810_b200 as lmcb
g = torch.Generator(device="cuda").manual_seed(1)
block = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ts = [(torch.randn(1024, 768, generator=g, device="cuda") * 0.02).to(torch.bfloat16),
      (torch.randn(3 * block, generator=g, device="cuda") * 0.02).to(torch.float16)]
codec = lmcb.Codec()
b = codec.compress(ts, block_size=block)
print([len(x) for x in b.to_bytes()])
