"""Shared-memory wavefronts per SASS instruction of one kernel from an ncu
report: totals per opcode and the instructions with the most excess
wavefronts.  usage  smem_conflicts.py REPORT KERNEL [top]"""
import csv, collections, subprocess, sys
path, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(['ncu', '-i', path, '-k', kernel, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; cur = None; seen = set(); ins = []
for r in rows:
    if 'Address' in r:
        hdr = r
        ia, isrc, iex = hdr.index('Address'), 3, hdr.index('Instructions Executed')
        iw, iwi = hdr.index('L1 Wavefronts Shared'), hdr.index('L1 Wavefronts Shared Ideal')
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] and r[0].isdigit():
        cur = (int(r[0]), r[1].strip()[:70])
        continue
    if not r[ia] or r[ia] in seen:
        continue
    seen.add(r[ia])
    try:
        ins.append((r[isrc], int(r[iex] or 0), int(r[iw] or 0), int(r[iwi] or 0), cur))
    except ValueError:
        pass
agg = collections.defaultdict(lambda: [0, 0, 0])
for s, ex, w, wi, c in ins:
    t = s.split()
    op = (t[1] if t[0].startswith('@') else t[0]).split('.')[0]
    if w:
        a = agg[op]; a[0] += ex; a[1] += w; a[2] += wi
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print('%-6s exec %.3fG wavefronts %.3fG ideal %.3fG' % (k, v[0] / 1e9, v[1] / 1e9, v[2] / 1e9))
byline = collections.defaultdict(lambda: [0, 0, 0])
for s, ex, w, wi, c in ins:
    if c and w > wi:
        a = byline[c]; a[0] += ex; a[1] += w; a[2] += wi
for c, v in sorted(byline.items(), key=lambda kv: -(kv[1][1] - kv[1][2]))[:top]:
    print('L%-5d excess %.3fG (exec %.3fG, %.2f wavefronts/inst) | %s' % (c[0], (v[1] - v[2]) / 1e9, v[0] / 1e9, v[1] / max(v[0], 1), c[1]))
