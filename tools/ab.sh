#!/bin/bash
# A/B per-kernel times: tools/ab.sh "cfg2 cfg4:delta" so1 so2 ... (LMCG_SERIAL=1: kernels one at a time)
cfgs=$1; shift
for so in "$@"; do
  cp $so paper_2505_09810_b200/liblmc_b200.so
  for c in $cfgs; do
    echo "== $so $c"; LMCG_SERIAL=1 python tools/ktime.py ${c%%:*} $( [[ $c == *:* ]] && echo ${c##*:} )
  done
done
