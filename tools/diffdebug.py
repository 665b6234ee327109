"""Debug helper: locate the first differing byte between the GPU stream and the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_09810_b200 as lmcb
from paper_2505_09810_b200 import synth
from oracle import oracle as O

def walk(stream):
    recs = []
    off = 28
    segs = int.from_bytes(stream[20:24], 'little')
    orig = int.from_bytes(stream[8:16], 'little')
    rem = orig
    while rem > 0:
        tab = [(int.from_bytes(stream[off+16*i:off+16*i+8],'little'), int.from_bytes(stream[off+16*i+8:off+16*i+16],'little')) for i in range(segs)]
        off += 16*segs
        for o, c in tab:
            end = off + c; p = off
            while p < end:
                mode = stream[p]; l = int.from_bytes(stream[p+1:p+5],'little')
                if mode == 1: ps = 1
                elif mode == 2: ps = l
                else: ps = 132 + (int.from_bytes(stream[p+5+128:p+5+132],'little')+7)//8
                recs.append((p, mode, l, ps)); p += 5 + ps
            off = end
        rem -= sum(o for o, _ in tab)
    return recs

codec = lmcb.Codec()
for cfg in sys.argv[1:]:
    specs, ts = synth.make_checkpoint(cfg, seed=1)
    b = codec.compress(ts)
    got = b.to_bytes()
    for i, t in enumerate(ts):
        raw = t.view(torch.uint8).reshape(-1).cpu().numpy().tobytes()
        want = O.compress(raw, 1, threads=8)
        g = got[i]
        if g == want:
            continue
        a = np.frombuffer(g, np.uint8); w = np.frombuffer(want, np.uint8)
        n = min(a.size, w.size)
        d = np.flatnonzero(a[:n] != w[:n])
        print(cfg, specs[i].name, 'len', len(g), len(want), 'ndiff', d.size, 'first', d[:10])
        if d.size:
            recs = walk(want)
            for p, mode, l, ps in recs:
                if p <= d[0] < p + 5 + ps:
                    print('  in record at', p, 'mode', mode, 'len', l, 'psize', ps, 'rel', d[0]-p)
                    bad_in = [(x - p) for x in d if p <= x < p+5+ps]
                    print('  diffs in this record rel:', bad_in[:20], 'count', len(bad_in))
                    break
            else:
                print('  header/table diff at', d[0])
            print('  got ', a[d[0]-4:d[0]+12]); print('  want', w[d[0]-4:d[0]+12])
        break
