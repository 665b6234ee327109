#!/bin/bash
# GPU box: GPU suite, then the bench lines of the delta / run-heavy configs (cfg4, cfg3) and cfg5 (with its delta step)
set -u
O=gpurun_out/$1; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/rc.log
tail -2 $O/pytest_gpu.log
for c in cfg4 cfg3 cfg5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" | tee -a $O/rc.log
  python - $O/bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); p=d['pipeline']
print(sys.argv[1], d['value'], 'c', p['compress_ms'], 'd', p['decompress_ms'], {k:v for k,v in d['kernels_ms_per_step'].items() if v>0.1})
ds=d.get('delta_step')
if ds: print('  delta step', ds['value'], 'c', ds['compress_gib_s'], 'd', ds['decompress_gib_s'], {k:v for k,v in ds['kernels_ms_per_step'].items() if v>0.3})
PY
done
