#!/bin/bash
# ncu --set full of the pair kernel's ASSIGN launch at C3 (fp16) and C4 (E5M2)
set -u
mkdir -p gpurun_out
for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $cfg
  timeout 300 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:assign_pair_kernel --launch-skip 4 -c 1 \
      -o gpurun_out/p_$1 timeout 900 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e \
      > gpurun_out/p_$1.log 2>&1
  echo "$1 ncu rc=$?"
done
