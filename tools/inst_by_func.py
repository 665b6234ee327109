import csv, collections, sys, subprocess, re
path = sys.argv[1]; src = sys.argv[2]
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if 'Address' in r)
hdr = rows[hi]; ia = hdr.index('Address'); iex = hdr.index('Instructions Executed'); ith=hdr.index('Thread Instructions Executed')
by = collections.Counter(); th=collections.Counter(); cur = None
for r in rows[hi + 1:]:
    if len(r) < len(hdr): continue
    if r[0] and r[0].isdigit():
        cur = int(r[0]); continue
    if cur is None or not r[ia]: continue
    try: by[cur] += int(r[iex] or 0); th[cur]+=int(r[ith] or 0)
    except ValueError: pass
# ranges from function starts in the source file
lines = open(src).read().split('\n')
starts = []
for i,l in enumerate(lines, 1):
    m = re.match(r'^(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?(\w+)\(', l)
    if m: starts.append((i, m.group(1)))
starts.append((len(lines)+1, 'END'))
tot = sum(by.values())
res=[]
for (a,n),(b,_) in zip(starts, starts[1:]):
    s_ = sum(v for k,v in by.items() if a<=k<b); t=sum(v for k,v in th.items() if a<=k<b)
    if s_: res.append((s_, n, a, t))
for s_,n,a,t in sorted(res, reverse=True)[:14]:
    print(f"{n:24s} L{a:5d} {s_/1e9:7.2f}G warp-inst {100*s_/tot:5.1f}%  thr/inst {t/max(s_,1):.1f}")
print('total', tot/1e9)
