#!/bin/bash
# fx_incr (segmented list, coalesced counts): FX tests, then per-iteration update times
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_virtual_ranks.py -q -x -k "fx or virtual" 2>&1 | tail -1
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; it=d['config']['lloyd_iters_per_step']; print('$1 $2', round(d['value']/1e12,3), 'e12; update us/iter', round(b['update']/it*1000,1), 'dist', round(b['dist']/it*1000,1))"; }
t c5_vq_10m fp16; t c5_vq_10m e5m2; t c3_blobs_1m_d64 fp16; t c4_blobs_1m_large e5m2
