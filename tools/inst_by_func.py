"""Instructions executed per source function from an ncu report (source page,
cuda+sass), per file: usage  inst_by_func.py REPORT [kernel-regex]"""
import csv, collections, os, re, subprocess, sys

path = sys.argv[1]
args = ['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass']
if len(sys.argv) > 2:
    args[3:3] = ['-k', sys.argv[2]]
rows = list(csv.reader(subprocess.run(args, capture_output=True, text=True).stdout.splitlines()))
by = collections.Counter(); th = collections.Counter()
cur_file, cur, hdr = None, None, None
for r in rows:
    if len(r) >= 2 and r[0] in ('File Name', 'File Path'):
        cur_file, cur = r[1], None
        continue
    if 'Address' in r:
        hdr = r; ia = hdr.index('Address'); iex = hdr.index('Instructions Executed')
        ith = hdr.index('Thread Instructions Executed')
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] and r[0].isdigit():
        cur = (cur_file, int(r[0]))
        continue
    if cur is None or not r[ia]:
        continue
    try:
        by[cur] += int(r[iex] or 0); th[cur] += int(r[ith] or 0)
    except ValueError:
        pass
tot = sum(by.values()) or 1
res = []
for f in sorted({k[0] for k in by}):
    if not f or not os.path.exists(f):
        continue
    lines = open(f).read().split('\n')
    starts = []
    for i, l in enumerate(lines, 1):
        m = re.match(r'^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__)[^(]*?(\w+)\(', l)
        if m:
            starts.append((i, m.group(1)))
    starts.append((len(lines) + 1, 'END'))
    for (a, n), (b, _) in zip(starts, starts[1:]):
        s_ = sum(v for (ff, k), v in by.items() if ff == f and a <= k < b)
        t = sum(v for (ff, k), v in th.items() if ff == f and a <= k < b)
        if s_:
            res.append((s_, f"{os.path.basename(f)}:{n}", a, t))
for s_, n, a, t in sorted(res, reverse=True)[:20]:
    print(f"{n:36s} L{a:5d} {s_/1e9:7.2f}G warp-inst {100*s_/tot:5.1f}%  thr/inst {t/max(s_,1):.1f}")
print('total', round(tot / 1e9, 3), 'G')
