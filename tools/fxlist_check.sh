#!/bin/bash
# changed-row listing by the distance kernel: FX / tc / virtual-rank / C5-scale tests, then the
# per-iteration update and distance times at C5 / C3 / C4 with and without it (interleaved)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_virtual_ranks.py tests/test_gpu_c5_scale.py -q -x 2>&1 | tail -2
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; it=d['config']['lloyd_iters_per_step']; print('$3 $1', round(d['value']/1e12,3), 'e12; update us/iter', round(b['update']/it*1000,1), 'dist', round(b['dist']/it*1000,1), 'clk', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
for cfg in "c5_vq_10m fp16" "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $cfg
  t $1 $2 listed; MPK_NO_FX_LIST=1 t $1 $2 fx_diff
done
done
