#!/bin/bash
# clock64 trace of the grouped one-tile path (trace build on the box)
mkdir -p gpurun_out
MPK_NVCC_EXTRA=-DMPK_PAIR_TRACE_RB=1 python __graft_entry__.py build > /dev/null 2>&1
for R in 4; do
MPK_PAIR_RBR=$R MPK_PAIR_TRACE=gpurun_out/trace_rbr_c4_$R.txt timeout 300 python bench.py --config c4_blobs_1m_large --dist e5m2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
MPK_PAIR_DBG=3 MPK_PAIR_RBR=$R MPK_PAIR_TRACE=gpurun_out/trace_rbr_c4_${R}_skel.txt timeout 300 python bench.py --config c4_blobs_1m_large --dist e5m2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
