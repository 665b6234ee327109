"""Opcode mix and per-loop instruction counts of one kernel from an ncu report
(SASS view): usage  sass_mix.py REPORT KERNEL [top]"""
import csv, collections, subprocess, sys
path, kernel = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(['ncu', '-i', path, '-k', kernel, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if 'Address' in r)
hdr = rows[hi]
ia, isrc, iex, ith = hdr.index('Address'), hdr.index('Source'), hdr.index('Instructions Executed'), hdr.index('Thread Instructions Executed')
ins = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[ia]:
        continue
    try:
        ins.append((r[ia], r[isrc], int(r[iex] or 0), int(r[ith] or 0)))
    except ValueError:
        pass
tot = sum(i[2] for i in ins) or 1
print('total warp-inst %.3fG over %d sass instructions' % (tot / 1e9, len(ins)))
ops = collections.Counter()
for a, s, ex, th in ins:
    t = s.split()
    op = t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '?')
    ops[op.split('.')[0]] += ex
print('opcode mix:', ', '.join('%s %.1f%%' % (o, 100 * c / tot) for o, c in ops.most_common(top)))
# runs of consecutive instructions with (nearly) equal execution counts = loops / phases
runs = []; cur = None
for idx, (a, s, ex, th) in enumerate(ins):
    if cur and ex > 0 and abs(ex - cur[2]) <= 0.02 * cur[2]:
        cur[1] = idx; cur[3] += ex
    else:
        if cur: runs.append(cur)
        cur = [idx, idx, ex, ex]
if cur: runs.append(cur)
for r in sorted(runs, key=lambda r: -r[3])[:top]:
    print('sass[%5d..%5d] n=%4d  exec/inst %.3fG  sum %.3fG %5.1f%%   %s' % (r[0], r[1], r[1] - r[0] + 1, r[2] / 1e9, r[3] / 1e9, 100 * r[3] / tot, ins[r[0]][1][:60]))
