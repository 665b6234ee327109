#!/bin/bash
# GPU box iteration: fused tests, GPU suite, cfg5 + cfg2 bench lines, ncu capture of one kernel on cfg5.
# usage: tools/iter.sh OUT [kernel-regex|-] [extra-test-args]
set -u
O=gpurun_out/$1; K=${2:--}
mkdir -p $O
timeout 240 python -m pytest tests/test_gpu_fused_decode.py -q -x > $O/pytest_fused.log 2>&1; echo "fused rc=$?" | tee -a $O/rc.log
tail -3 $O/pytest_fused.log
grep -q "fused rc=0" $O/rc.log || exit 1
timeout 600 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/rc.log
tail -3 $O/pytest_gpu.log
for c in cfg5 cfg2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?" | tee -a $O/rc.log
  python - $O/bench_$c.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); p=d['pipeline']
print(sys.argv[1], d['value'], 'c', p['compress_ms'], 'd', p['decompress_ms'], {k:v for k,v in d['kernels_ms_per_step'].items() if v>0.05})
PY
done
if [ "$K" != "-" ]; then
  CONFIG=cfg5 bash tools/profile_kernel.sh $K 1
  mv gpurun_out/prof_k.ncu-rep $O/$K.ncu-rep 2>/dev/null
fi
