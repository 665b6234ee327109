"""Summarise gpurun_out ncu artefacts into profiles/ (launch list shares + full-capture metrics)."""
import collections
import csv
import json
import os
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[hi]
    ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
            continue
        name = r[ki].split('(')[0].split()[-1]
        v = float(r[vi].replace(',', ''))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": c, "total_ns": round(t), "avg_us": round(t / c / 1e3, 2), "share": round(t / tot, 4)}
            for k, (c, t) in agg.items()}


def full(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread',
            'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
            'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
            'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size', 'smsp__inst_executed.sum',
            'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
    res = {}
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')].split('(')[0]
        res[name] = {w: r[hdr.index(w)] + ' ' + units[hdr.index(w)] for w in want if w in hdr}
    return res


def to_bytes(s):
    v, u = s.split()
    return float(v) * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}[u]


if __name__ == '__main__':
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else 'gpurun_out'
    res = {}
    if os.path.exists(f'{src}/launches.csv'):
        res['launch_list'] = launches(f'{src}/launches.csv')
    if os.path.exists(f'{src}/prof.ncu-rep'):
        res['full'] = full(f'{src}/prof.ncu-rep')
        traffic = {k: to_bytes(d['dram__bytes_read.sum']) + to_bytes(d['dram__bytes_write.sum'])
                   for k, d in res['full'].items()}
        res['traffic_bytes_per_launch'] = traffic
        cfg = os.environ.get('CONFIG', 'cfg2')
        try:
            allt = json.load(open('profiles/ncu_traffic.json'))
            if not all(isinstance(v, dict) for v in allt.values()):
                allt = {}
        except Exception:
            allt = {}
        allt[cfg] = traffic
        json.dump(allt, open('profiles/ncu_traffic.json', 'w'), indent=1)
    json.dump(res, open(f'profiles/{tag}_ncu.json', 'w'), indent=1)
    print(json.dumps(res.get('launch_list', {}), indent=1))
