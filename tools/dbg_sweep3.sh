#!/bin/bash
# 0 full; 16 full with one reused X~ tile (no HBM stream); 17 MMAs only + reused tile;
# 1 MMAs only; 19 handshakes only + reused tile
for dbg in 0 16 17 1 19; do
  MPK_PAIR_DBG=$dbg timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist fp16 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('dbg=$dbg', round(d['roofline']['avg_launch_ms'],3), 'ms')"
done
