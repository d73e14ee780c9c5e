#!/bin/bash
# launch times of the pair kernel at C3 / C4 / C5 for compile-time variants (MPK_NVCC_EXTRA)
mkdir -p gpurun_out
for v in "" "-DMPK_PAIR_WAIT2=0" "-DMPK_PAIR_MMA2=0" "-DMPK_PAIR_WAIT2=0 -DMPK_PAIR_MMA2=0" "-DMPK_WAIT_TRY=1" "-DMPK_WAIT_TRY=1 -DMPK_PAIR_WAIT2=0"; do
  MPK_NVCC_EXTRA="$v -DMPK_VARIANT_TAG" python __graft_entry__.py build > /dev/null 2>&1 || echo "build failed: $v"
  for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2" "c5_vq_10m fp16" "c5_vq_10m e5m2"; do
    set -- $cfg
    timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('[$v] $1 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us', 'clk', d['clocks']['sm_mhz'])"
  done
done
