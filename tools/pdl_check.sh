#!/bin/bash
# programmatic dependent launch (update chain, finalize, centroid prep, distance kernel) and the
# memsets folded into finalize: tests, then per-iteration times with and without PDL
timeout 2000 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; it=d['config']['lloyd_iters_per_step']; print('$3 $1 $2', round(d['value']/1e12,4), 'e12; it/s', round(d['lloyd_iters_per_s']), 'update', round(b['update']/it*1000,1), 'dist', round(b['dist']/it*1000,1), 'loop ms', round(b['loop'],3))"; }
for rep in 1 2; do
for cfg in "c4_blobs_1m_large e5m2" "c3_blobs_1m_d64 fp16" "c5_vq_10m fp16"; do
  set -- $cfg
  t $1 $2 pdl; MPK_NO_PDL=1 t $1 $2 plain
done
done
