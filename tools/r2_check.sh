#!/bin/bash
# GPU box: the parity suite, smoke, the default bench line (cfg5) and the reference arm.
set -u
O=gpurun_out/${1:-r2}
mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/rc.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/rc.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/rc.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" | tee -a $O/rc.log
