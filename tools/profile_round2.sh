#!/bin/bash
# Round-2 evidence for profiles/: measured FP8 peak, GPU tests + smoke, bench lines (fp16 and
# E5M2, both arms), the ncu launch list of the bench command, and one ncu --set full capture of
# the distance kernel per operand format with the tensor-pipe metrics added. Each ncu pass runs
# only after the same command exited 0 without ncu. Usage: tools/profile_round2.sh <tag> [skip-tests]
set -u
tag=${1:-round2}
mkdir -p gpurun_out profiles
TP=sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tmem.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 python tools/measure_fp8_peak.py --out gpurun_out/fp8_peak.json > gpurun_out/${tag}_fp8_peak.log 2>&1
echo "fp8 peak rc=$?"
[ -s gpurun_out/fp8_peak.json ] && cp gpurun_out/fp8_peak.json profiles/fp8_peak.json
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${tag}_gpu_tests.log 2>&1
  echo "gpu tests rc=$?"
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
  echo "smoke rc=$?"
fi
timeout 900 python bench.py > gpurun_out/${tag}_bench_c5_fp16.json 2> gpurun_out/${tag}_bench_c5_fp16.err; rc=$?
echo "bench fp16 rc=$rc"
timeout 900 python bench.py --dist e5m2 > gpurun_out/${tag}_bench_c5_e5m2.json 2> gpurun_out/${tag}_bench_c5_e5m2.err
echo "bench e5m2 rc=$?"
MPK_PAIR_DBG=1 timeout 600 python bench.py --dist e5m2 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_c5_e5m2_mma_only.json 2>&1
echo "bench e5m2 mma-only rc=$?"
MPK_PAIR_DBG=1 timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_c5_fp16_mma_only.json 2>&1
echo "bench fp16 mma-only rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_reference_c5.json 2> gpurun_out/${tag}_bench_ref.err
echo "reference rc=$?"
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
