#!/bin/bash
# rbh with 2 vs 4 parts (accumulators) per warpgroup: parity subset and C5 launch times
t() { MPK_PAIR_DBG=$3 timeout 300 python bench.py --dist $1 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$2 $1 dbg=$3', round(d['roofline']['avg_launch_ms']*1000,1), 'us clk', d['clocks']['sm_mhz'])"; }
for P in 4 2; do
  MPK_NVCC_EXTRA="-DMPK_PAIR_RBH_PARTS=$P" python __graft_entry__.py build > /dev/null 2>&1 || echo "build failed $P"
  timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_c5_scale.py -q -x -k "halves or deep_row_blocks_c5 or matches_oracle or teacher or final" 2>&1 | tail -1
  t fp16 "P=$P" 0; t fp16 "P=$P" 0; t fp16 "P=$P" 1; t e5m2 "P=$P" 0
done
