#!/bin/bash
set -u
for spec in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $spec
  for dbg in 0 3 11 19 27 1 9 17; do
    MPK_PAIR_DBG=$dbg timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 dbg=$dbg', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
  done
done
