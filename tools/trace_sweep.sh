#!/bin/bash
# per-tile clock64 trace of the pair kernel's leader CTA at C5 fp16 for the given debug modes
mkdir -p gpurun_out
for dbg in "$@"; do
  MPK_PAIR_DBG=$dbg MPK_PAIR_TRACE=gpurun_out/trace_$dbg.txt timeout 300 python bench.py --steps 1 --warmup 3 --iters 2 --dist ${DIST:-fp16} --no-cpu-baseline --no-e2e > /dev/null 2>gpurun_out/trace_err_$dbg.txt
  echo "dbg=$dbg rc=$?"
  MPK_PAIR_DBG=$dbg timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist ${DIST:-fp16} --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('dbg=$dbg', round(d['roofline']['avg_launch_ms'],3), 'ms')"
done
