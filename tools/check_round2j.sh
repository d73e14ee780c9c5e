#!/bin/bash
set -u
tag=${1:-round2j}
mkdir -p gpurun_out
for dbg in 0 4 2 6; do
  MPK_PAIR_DBG=$dbg timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 fp16 dbg=$dbg', round(d['roofline']['avg_launch_ms'],4), 'ms', d['clocks']['sm_mhz'])"
done
for nb in 256 128; do
  MPK_PAIR_NB=$nb timeout 300 python bench.py --config c3_blobs_1m_d64 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c3 nb=$nb', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
done
