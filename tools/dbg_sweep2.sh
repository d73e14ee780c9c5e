#!/bin/bash
# Pair-kernel decomposition (C5 fp16, NB=256): 0 full; 2 no MMA; 2+4 TMEM loads only;
# 2+8 fold only (no TMEM loads); 1 no epilogue; 3 handshakes only.
for dbg in 0 2 6 10 1 3; do
  MPK_PAIR_DBG=$dbg timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist fp16 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('dbg=$dbg', round(d['roofline']['avg_launch_ms'],3), 'ms')"
done
