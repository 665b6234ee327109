#!/bin/bash
# A/B of built library variants on the GPU box: tools/ab.sh "cfg2 cfg5" a.so b.so ...
# Per variant and config: bench value, compress / decompress ms (graphs, side
# stream on), then the per-kernel times with LMCG_SERIAL=1 (kernels one at a time).
cfgs=$1; shift
for so in "$@"; do
  cp $so paper_2505_09810_b200/liblmc_b200.so
  for c in $cfgs; do
    for ser in 0 1; do
      LMCG_SERIAL=$ser python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['pipeline']; print('$so $c serial=$ser', d['value'], 'c', p['compress_ms'], 'd', p['decompress_ms'], {k: v for k, v in d['kernels_ms_per_step'].items() if v > 0.05} if $ser else '')"
    done
  done
done
