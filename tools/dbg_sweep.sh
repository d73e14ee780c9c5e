#!/bin/bash
# Per-tile cost decomposition of the pair kernel (C5, fp16): normal, no epilogue folding, no MMAs.
for nb in 128 256; do
  for dbg in 0 1 2 3; do
    MPK_PAIR_NB=$nb MPK_PAIR_DBG=$dbg timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist fp16 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('NB=$nb dbg=$dbg', round(d['roofline']['avg_launch_ms'],3), 'ms')"
  done
done
