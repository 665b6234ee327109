#!/bin/bash
# GPU box: decompress time per config with fusion forced on / off.
set -u
O=gpurun_out/${1:-fab}; mkdir -p $O
timeout 240 python -m pytest tests/test_gpu_fused_decode.py -q -x 2>&1 | tail -1
for c in ${CFGS:-cfg1 cfg2 cfg3 cfg4 cfg5}; do
  for mode in on off; do
    if [ $mode = on ]; then export LMCG_FUSE_FROM=0; unset LMCG_NOFUSE; else export LMCG_NOFUSE=1; unset LMCG_FUSE_FROM; fi
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/$c.$mode.json 2> $O/$c.$mode.err
    python - $O/$c.$mode.json $c $mode <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); p=d['pipeline']
    print(sys.argv[2], sys.argv[3], d['value'], 'c', p['compress_ms'], 'd', p['decompress_ms'])
except Exception as e: print(sys.argv[2], sys.argv[3], 'failed', e)
PY
  done
done
