#!/bin/bash
# Round-2: small-d K5g pipelined, seeding prefetch; C3/C4 pair-kernel captures.
set -u
tag=${1:-round2c}
mkdir -p gpurun_out
TP=sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 python -m pytest tests/test_gpu_seed.py tests/test_gpu_parity.py tests/test_gpu_image_sweep.py -q -m gpu -x > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
for cfg in c2_image_512 c2_image_4096; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err; echo "bench $cfg rc=$?"
done
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/${tag}_bench_seed.json 2>&1; echo "seed rc=$?"
for cfg in c3_blobs_1m_d64 c4_blobs_1m_large; do
  ncu --set full --metrics $TP --import-source on --clock-control none -k regex:assign_pair_kernel --launch-skip 4 -c 1 \
      -o gpurun_out/${tag}_pair_${cfg} timeout 600 python bench.py --config $cfg --steps 1 --warmup 3 --iters 2 \
      --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_${cfg}.log 2>&1
  echo "ncu $cfg rc=$?"
done
ncu --set full --import-source on --clock-control none -k regex:smalld_iter --launch-skip 30 -c 1 \
    -o gpurun_out/${tag}_smalld_4096 timeout 600 python bench.py --config c2_image_4096 --steps 1 --warmup 3 --iters 4 \
    --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_smalld.log 2>&1
echo "ncu smalld rc=$?"
