#!/bin/bash
# Round measurement on the GPU box: tests, the bench line (both arms), every
# config, chain + pipeline benches, torchrun N=1, ncu launch list and full
# captures (cfg2, cfg5).  Output: gpurun_out/final/
set -u
O=gpurun_out/${1:-final}
mkdir -p $O/configs
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/rc.log
python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/rc.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/rc.log
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" | tee -a $O/rc.log
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/configs/$c.json 2> $O/configs/$c.err; echo "$c rc=$?" | tee -a $O/rc.log
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $O/configs/${c}_ref.json 2> $O/configs/${c}_ref.err; echo "$c ref rc=$?" | tee -a $O/rc.log
done
timeout 900 python tools/bench_chain.py > $O/configs/chain.json 2> $O/configs/chain.err; echo "chain rc=$?" | tee -a $O/rc.log
for c in cfg2 cfg4; do
  timeout 900 python tools/bench_pipeline.py --config $c > $O/configs/pipeline_$c.json 2> $O/configs/pipeline_$c.err; echo "pipeline $c rc=$?" | tee -a $O/rc.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > $O/torchrun1.json 2> $O/torchrun1.err; echo "torchrun rc=$?" | tee -a $O/rc.log
# ncu: launch list (cfg2 default bench command), full captures of the hot kernels (cfg2, cfg5)
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py $ARGS > $O/ncu_launch.log 2>&1; echo "launch rc=$?" | tee -a $O/rc.log
for c in cfg2 cfg5; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_decrec|k_encode|k_hist|k_decpair|k_crc|k_ungroup|k_codebook|k_cand" -c 7 -o $O/prof_$c python bench.py $ARGS --config $c > $O/ncu_full_$c.log 2>&1; echo "full $c rc=$?" | tee -a $O/rc.log
done
