#!/bin/bash
# GPU box: gpu tests, cfg2 summary (tools/quick.sh) and short cfg5 / cfg4 kernel tables
bash tools/quick.sh
for c in ${CFGS:-cfg5}; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['pipeline']); print({k: v for k, v in d['kernels_ms_per_step'].items() if v > 0.05})"
done
