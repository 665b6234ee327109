import csv, collections, sys, subprocess
path = sys.argv[1]
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if 'Address' in r)
hdr = rows[hi]; ia = hdr.index('Address'); iex = hdr.index('Instructions Executed'); ith=hdr.index('Thread Instructions Executed')
ifile = None
by = collections.Counter(); th=collections.Counter(); cur = None; curfile=None
for r in rows[hi + 1:]:
    if len(r) < len(hdr): continue
    if r[0] and r[0].isdigit():
        cur = int(r[0]); continue
    if cur is None or not r[ia]: continue
    try: by[cur] += int(r[iex] or 0); th[cur]+=int(r[ith] or 0)
    except ValueError: pass
ranges = [(300,336,'step1/Src'),(337,375,'decode_span setup/adv'),(376,487,'pass0 bitmap+checkpoints+fix'),(488,505,'emit head'),(506,599,'bulk loop (count+emit)'),(600,697,'huff_passes'),(698,807,'huff_decode setup'),(808,876,'LUT builds'),(877,939,'copy/decode_record'),(1396,1425,'plane16/crc_word'),(1426,1545,'k_decpair body')]
tot = sum(by.values())
for a,b,n in ranges:
    s = sum(v for k,v in by.items() if a<=k<=b); t=sum(v for k,v in th.items() if a<=k<=b)
    print(f"{n:32s} {s/1e9:7.2f}G warp-inst {100*s/tot:5.1f}%  thr/inst {t/max(s,1):.1f}")
other = sum(v for k,v in by.items() if not any(a<=k<=b for a,b,_ in ranges))
print('other', other/1e9, 'total', tot/1e9)
top_other = sorted(((v,k) for k,v in by.items() if not any(a<=k<=b for a,b,_ in ranges)), reverse=True)[:8]
print(top_other)
