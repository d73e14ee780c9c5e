#!/bin/bash
# labels vs oracle (tc_check) + pair-kernel timing at C5 for fp16/e5m2 + per-tile trace
mkdir -p gpurun_out
timeout 300 python tools/tc_check.py 2>&1 | tail -12
for dist in fp16 e5m2 bf16; do
  timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist $dist --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$dist', round(d['roofline']['avg_launch_ms'],3), 'ms', round(d['roofline']['frac'],3), d['value'])"
done
for dbg in 0; do
  MPK_PAIR_DBG=$dbg MPK_PAIR_TRACE=gpurun_out/trace_$dbg.txt timeout 300 python bench.py --steps 1 --warmup 3 --iters 2 --dist fp16 --no-cpu-baseline --no-e2e > /dev/null
done
