#!/bin/bash
# GPU box: gpu tests (short), bench summary line, optional debug counters.
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['pipeline']); print({k: v for k, v in d['kernels_ms_per_step'].items() if v > 0.015})"
if [ "${1:-}" = dbg ]; then python tools/debug_counters.py cfg2 2>&1 | grep -E "cyc|rounds|recs|fix"; fi
