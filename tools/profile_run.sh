#!/bin/bash
# Run on the GPU box (under gpurun): plain bench, launch list, one full capture per hot kernel.
set -u
OUT=${1:-gpurun_out}
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline --config ${CONFIG:-cfg2}"
mkdir -p $OUT
timeout 300 python bench.py $ARGS > $OUT/prof_plain.log 2>&1 || { echo "plain run failed"; tail -20 $OUT/prof_plain.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decrec|k_encode|k_hist|k_decpair|k_crc|k_ungroup|k_codebook|k_cand|k_frame|k_finalize" -c 9 -o $OUT/prof python bench.py $ARGS > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
ls -la $OUT
