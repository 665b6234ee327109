#!/bin/bash
# GPU box: one ncu --set full capture of kernel $2 on config $3 (default cfg5) into gpurun_out/$1/
set -u
O=gpurun_out/$1; K=$2; mkdir -p $O
CONFIG=${3:-cfg5} bash tools/profile_kernel.sh $K 1
mv gpurun_out/prof_k.ncu-rep $O/$K.ncu-rep 2>/dev/null
