#!/bin/bash
# GPU box: decode phase counters (debug build) on cfg5 and one ncu --set full capture of k_decpair.
set -u
O=gpurun_out/${1:-pp}
mkdir -p $O
timeout 600 python tools/debug_counters.py cfg5 > $O/dbg_cfg5.txt 2>&1; echo "dbg rc=$?"
CONFIG=cfg5 bash tools/profile_kernel.sh k_decpair 1
mv gpurun_out/prof_k.ncu-rep $O/decpair_cfg5.ncu-rep 2>/dev/null
tail -3 gpurun_out/ncu_k.log
