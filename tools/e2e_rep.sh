#!/bin/bash
# GPU box: repeat the default bench (with e2e) to catch intermittent decode errors.
for i in $(seq 1 ${1:-4}); do
  timeout 300 python bench.py --config ${CFG:-cfg5} --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e$i.json 2> gpurun_out/e$i.err; echo "run $i rc=$? $(tail -1 gpurun_out/e$i.err | cut -c1-250)"
done
