#!/bin/bash
# Round-2 evidence: GPU tests + smoke, the default bench line (C5 fp16) and E5M2, the reference
# arm, supplementary lines (C2 512^2 / 4096^2, C3, C4, delta = 2, D^2 seeding), the ncu launch
# list and full captures (tensor-pipe metrics) of the distance kernel.
set -u
tag=${1:-round2z}
mkdir -p gpurun_out
TP=sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${tag}_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${tag}_bench_c5_fp16.json 2> gpurun_out/${tag}_bench_c5_fp16.err; rc=$?; echo "bench rc=$rc"
timeout 900 python bench.py --dist e5m2 > gpurun_out/${tag}_bench_c5_e5m2.json 2> gpurun_out/${tag}_bench_c5_e5m2.err; echo "e5m2 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_reference_c5.json 2> gpurun_out/${tag}_bench_ref.err; echo "ref rc=$?"
for cfg in c2_image_512 c2_image_4096 c3_blobs_1m_d64 c4_blobs_1m_large c1_blobs_small; do
  timeout 600 python bench.py --config $cfg --no-e2e > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err; echo "$cfg rc=$?"
done
timeout 900 python bench.py --delta 2 --steps 3 --iters 5 --no-e2e > gpurun_out/${tag}_bench_delta2_c5.json 2>&1; echo "delta rc=$?"
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/${tag}_bench_seed_d2_c5.json 2>&1; echo "seed rc=$?"
if [ $rc -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c5_fp16.csv \
      timeout 1200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_launch.log 2>&1
  echo "launch list rc=$?"
  for dist in fp16 e5m2; do
    ncu --set full --metrics $TP --import-source on --clock-control none -k regex:assign_pair_kernel --launch-skip 4 -c 1 \
        -o gpurun_out/${tag}_pair_full_${dist} timeout 900 python bench.py --dist $dist --steps 1 --warmup 3 --iters 2 \
        --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_full_${dist}.log 2>&1
    echo "full capture $dist rc=$?"
  done
fi
