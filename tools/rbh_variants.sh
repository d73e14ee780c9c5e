#!/bin/bash
# rbh variants (compile-time): C5 fp16 distance launch times
t() { MPK_PAIR_DBG=$3 timeout 300 python bench.py --dist $1 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$2 $1 dbg=$3', round(d['roofline']['avg_launch_ms']*1000,1), 'us clk', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for v in "" "-DMPK_PAIR_RBH_STAGGER=4" "-DMPK_PAIR_RBH_STAGGER=1"; do
  MPK_NVCC_EXTRA="$v -DMPK_VARIANT" python __graft_entry__.py build > /dev/null 2>&1 || echo "build failed $v"
  t fp16 "[$v]" 0
done
done
