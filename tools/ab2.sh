#!/bin/bash
# A/B of library variants: tools/ab2.sh "cfg5" var_so/a.so var_so/b.so ... (serial and overlapped compress timings)
cfgs=$1; shift
cp paper_2505_09810_b200/liblmc_b200.so /tmp/keep.so
for so in "$@"; do
  cp $so paper_2505_09810_b200/liblmc_b200.so
  for c in $cfgs; do
    for ser in 0 1; do
      LMCG_SERIAL=$ser timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['pipeline']; print('$so $c serial=$ser', d['value'], 'c', p['compress_ms'], 'd', p['decompress_ms'], {k: v for k, v in d['kernels_ms_per_step'].items() if v > 0.3} if $ser else '')"
    done
  done
done
cp /tmp/keep.so paper_2505_09810_b200/liblmc_b200.so
