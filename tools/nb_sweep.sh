#!/bin/bash
# Sweep the pair kernel's centroid tile width on the C5 workload (distance kernel ms per launch).
for nb in 64 128 256; do
  for dd in fp16 e5m2; do
    MPK_PAIR_NB=$nb timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist $dd --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('NB=$nb', '$dd', round(d['roofline']['avg_launch_ms'],3), 'ms', round(d['roofline']['frac'],3))"
  done
done
