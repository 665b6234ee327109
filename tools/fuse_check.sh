#!/bin/bash
# GPU box: fused-decode tests, the GPU suite, and cfg5/cfg2 bench lines with fusion on and off.
set -u
O=gpurun_out/${1:-fuse}
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fused_decode.py -q -x > $O/pytest_fused.log 2>&1; echo "fused rc=$?" | tee -a $O/rc.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/rc.log
for c in cfg5 cfg2; do
  for f in 0 1; do
    LMCG_NOFUSE=$f timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_${c}_nofuse$f.json 2> $O/bench_${c}_nofuse$f.err; echo "bench $c nofuse=$f rc=$?" | tee -a $O/rc.log
  done
done
