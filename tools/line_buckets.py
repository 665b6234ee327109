"""Instructions executed per source line (ncu source page), for one kernel: python tools/line_buckets.py rep kernel [min%]"""
import subprocess, csv, collections, sys
rep, kern = sys.argv[1], sys.argv[2]
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass', '-k', kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if 'Address' in r); hdr = rows[hi]
ia = hdr.index('Address'); iex = hdr.index('Instructions Executed')
cur = None; per = collections.Counter(); src = {}
for r in rows[hi + 1:]:
    if len(r) < len(hdr): continue
    if r[0] and r[0].isdigit(): cur = int(r[0]); src[cur] = r[1][:90]; continue
    if cur is None or not r[ia]: continue
    try: per[cur] += float(r[iex] or 0)
    except ValueError: pass
tot = sum(per.values())
print('total warp instructions', int(tot))
for l, v in sorted(per.items()):
    if 100 * v / tot >= mn: print(f"L{l:5d} {100 * v / tot:5.1f}%  {src.get(l, '')}")
