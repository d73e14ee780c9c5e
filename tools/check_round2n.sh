#!/bin/bash
set -u
for dist in fp16 e5m2; do
  for dbg in 0 1 2 3 11 27; do
    MPK_PAIR_DBG=$dbg timeout 300 python bench.py --dist $dist --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 $dist dbg=$dbg', round(d['roofline']['avg_launch_ms']*1e3,1), 'us', d['clocks']['sm_mhz'])"
  done
done
