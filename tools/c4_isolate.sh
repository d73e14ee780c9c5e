#!/bin/bash
# distance launch times at C4 / C3 / C5 (current build)
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 $1 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us clk', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  t c4_blobs_1m_large e5m2 list; MPK_NO_FX_LIST=1 t c4_blobs_1m_large e5m2 nolist
  t c3_blobs_1m_d64 fp16 list; t c5_vq_10m fp16 list; t c5_vq_10m e5m2 list
done
