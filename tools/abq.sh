#!/bin/bash
# A/B of whole-pipeline bench numbers (overlap on): tools/abq.sh "cfg2 cfg5" so1 so2 ...
cfgs=$1; shift
for so in "$@"; do
  cp $so paper_2505_09810_b200/liblmc_b200.so
  for c in $cfgs; do
    python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['pipeline']; print('$(basename $so)', '$c', d['value'], p['compress_ms'], p['decompress_ms'])"
  done
done
