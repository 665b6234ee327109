"""gpurun_out/<run> ncu artefacts -> profiles/<dest>/ summaries and profiles/ncu_traffic.json.
usage: summarize_round.py RUN_DIR DEST_DIR"""
import json, os, shutil, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import full, launches, to_bytes   # noqa: E402

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)
if os.path.exists(f'{src}/launches.csv'):
    json.dump(launches(f'{src}/launches.csv'), open(f'{dst}/launch_list_cfg5.json', 'w'), indent=1)
    shutil.copy(f'{src}/launches.csv', f'{dst}/launches.csv')
allt = json.load(open('profiles/ncu_traffic.json'))
for cfg in ('cfg2', 'cfg5'):
    p = f'{src}/prof_{cfg}.ncu-rep'
    if not os.path.exists(p):
        continue
    res = full(p)
    json.dump(res, open(f'{dst}/ncu_summary_{cfg}.json', 'w'), indent=1)
    allt[cfg] = {k: to_bytes(d['dram__bytes_read.sum']) + to_bytes(d['dram__bytes_write.sum']) for k, d in res.items()}
json.dump(allt, open('profiles/ncu_traffic.json', 'w'), indent=1)
for f in ('bench.json', 'bench_ref.json', 'pytest_gpu.log', 'smoke.log', 'torchrun1.json', 'rc.log'):
    if os.path.exists(f'{src}/{f}'):
        shutil.copy(f'{src}/{f}', f'{dst}/{f}')
if os.path.isdir(f'{src}/configs'):
    shutil.copytree(f'{src}/configs', f'{dst}/configs', dirs_exist_ok=True)
print(json.dumps(allt, indent=1))
