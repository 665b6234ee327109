#!/bin/bash
# GPU box: failure rate of back-to-back plan replays under a few switches
N=${1:-600}
echo "== base"; timeout 300 python tools/stress.py cfg5 $N 2>&1 | tail -4
echo "== no eager pass"; STRESS_NOEAGER=1 timeout 300 python tools/stress.py cfg5 $N 2>&1 | tail -4
echo "== no fusion"; STRESS_NOFUSE=1 timeout 300 python tools/stress.py cfg5 $N 2>&1 | tail -4
echo "== base again"; timeout 300 python tools/stress.py cfg5 $N 2>&1 | tail -4
