#!/bin/bash
# usage: tools/profile_kernel.sh <kernel-regex> [count]  (run under gpurun)
set -u
K=$1; C=${2:-1}
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --config ${CONFIG:-cfg2}"
mkdir -p gpurun_out
timeout 300 python bench.py $ARGS > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/prof_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c $C -o gpurun_out/prof_k python bench.py $ARGS > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?"
