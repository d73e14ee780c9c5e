#!/bin/bash
# parity subset + launch times (normal build), then fine clock64 stamps of the pair kernel's MMA
# loop (trace build on the box) at C4 / C3
mkdir -p gpurun_out
bash tools/roles_check.sh
MPK_NVCC_EXTRA=-DMPK_PAIR_TRACE_RB=1 python __graft_entry__.py build > /dev/null 2>&1
for cfg in "c4_blobs_1m_large e5m2" "c3_blobs_1m_d64 fp16"; do
  set -- $cfg
  MPK_PAIR_TRACE=gpurun_out/trace_mma_${1}.txt timeout 300 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
