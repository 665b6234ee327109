#!/bin/bash
# Every BASELINE.json config through bench.py, both arms (GPU box): gpurun_out/cfgs/
mkdir -p gpurun_out/cfgs
for c in ${CONFIGS:-cfg1 cfg2 cfg3 cfg4 cfg5}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfgs/$c.json 2> gpurun_out/cfgs/$c.err
  echo "$c ours rc=$?"
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/cfgs/${c}_ref.json 2> gpurun_out/cfgs/${c}_ref.err
  echo "$c ref rc=$?"
done
