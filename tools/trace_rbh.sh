#!/bin/bash
# clock64 trace of the rbh path at C5 fp16 (trace build on the box): full and MMA-only
mkdir -p gpurun_out
MPK_NVCC_EXTRA=-DMPK_PAIR_TRACE_RB=1 python __graft_entry__.py build > /dev/null 2>&1
for dbg in 0 1; do
  MPK_PAIR_DBG=$dbg MPK_PAIR_TRACE=gpurun_out/trace_rbh_$dbg.txt timeout 300 python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
