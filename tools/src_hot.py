"""Aggregate an ncu source page (cuda,sass) by CUDA line: instructions, active threads, stalls."""
import csv, collections, sys
path, kernel = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
import subprocess
args = ['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass']
if kernel: args[3:3] = ['-k', kernel]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if 'Address' in r)
hdr = rows[hi]
ia = hdr.index('Address'); iex = hdr.index('Instructions Executed'); ith = hdr.index('Thread Instructions Executed')
ist = hdr.index('Warp Stall Sampling (All Samples)')
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
by = collections.defaultdict(lambda: collections.Counter()); src = {}; cur = None
for r in rows[hi + 1:]:
    if len(r) < len(hdr): continue
    if r[0] and r[0].isdigit():
        cur = int(r[0]); src[cur] = r[1][:95]
        continue
    if cur is None or not r[ia]: continue
    c = by[cur]
    try:
        c['ex'] += int(r[iex] or 0); c['th'] += int(r[ith] or 0); c['st'] += int(r[ist] or 0)
        for h in stalls: c[h] += int(r[hdr.index(h)] or 0)
    except ValueError:
        pass
tex = sum(c['ex'] for c in by.values()) or 1; tst = sum(c['st'] for c in by.values()) or 1
agg = collections.Counter()
for c in by.values():
    for h in stalls: agg[h] += c[h]
print('warp instructions', tex, 'stall mix', {k[6:]: round(v / tst * 100, 1) for k, v in agg.most_common(8)})
key = sys.argv[3] if len(sys.argv) > 3 else 'ex'
for ln, c in sorted(by.items(), key=lambda kv: -kv[1][key])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    top = [h[6:] for h, _ in collections.Counter({h: c[h] for h in stalls}).most_common(2)]
    print(f"L{ln:4d} {c['ex']/tex*100:5.1f}%inst {c['st']/tst*100:5.1f}%stall thr={c['th']/max(c['ex'],1):4.1f} {top} | {src.get(ln,'')}")
