#!/bin/bash
# per-tile clock64 trace of the pair kernel's leader CTA at C3 (fp16) and C4 (E5M2), plus the
# launch time, for the given debug modes (MPK_PAIR_DBG)
mkdir -p gpurun_out
for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $cfg
  for dbg in 0 3 27; do
    MPK_PAIR_DBG=$dbg MPK_PAIR_TRACE=gpurun_out/trace_${1}_$dbg.txt timeout 300 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>gpurun_out/trace_err_${1}_$dbg.txt
    MPK_PAIR_DBG=$dbg timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 dbg=$dbg', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"
  done
done
