#!/bin/bash
# compress time with k_crc forked before / after the histogram
for f in 0 1; do for c in cfg2 cfg5; do
LMCG_CRC_FORK=$f python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fork$f $c', d['value'], d['pipeline']['compress_ms'], d['pipeline']['decompress_ms'])"
done; done
