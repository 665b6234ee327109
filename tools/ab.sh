#!/bin/bash
# A/B per-kernel times: tools/ab.sh cfg so1 so2 ... (serial kernels, LMCG_SERIAL=1)
cfg=$1; shift
for so in "$@"; do
  cp $so paper_2505_09810_b200/liblmc_b200.so
  echo "== $so"; LMCG_SERIAL=1 python tools/ktime.py $cfg; python tools/ktime.py $cfg
done
