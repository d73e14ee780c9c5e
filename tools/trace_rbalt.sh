#!/bin/bash
# clock64 trace of the row-block alternation at C3 / C4 (a trace build on the box), and C4 with
# MPK_PAIR_DBG=8 (no X~ loads) timed on the normal build
mkdir -p gpurun_out
for cfg in "c4_blobs_1m_large e5m2" "c3_blobs_1m_d64 fp16"; do
  set -- $cfg
  for dbg in 0 8; do
  MPK_PAIR_DBG=$dbg timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $2 dbg=$dbg', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"
  done
done
MPK_NVCC_EXTRA=-DMPK_PAIR_TRACE_RB=1 python __graft_entry__.py build > /dev/null 2>&1
for cfg in "c4_blobs_1m_large e5m2" "c3_blobs_1m_d64 fp16"; do
  set -- $cfg
  MPK_PAIR_TRACE=gpurun_out/trace_rb2_${1}.txt timeout 300 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
