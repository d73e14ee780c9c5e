#!/bin/bash
# Round-2 iteration check: the GPU tests touched by this change set, then the supplementary
# bench lines (C2 512^2 and 4096^2 images, C3, C4, D^2 seeding at C5, a short C5 line).
set -u
tag=${1:-round2b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_seed.py tests/test_gpu_parity.py tests/test_gpu_image_sweep.py tests/test_gpu_virtual_ranks.py tests/test_gpu_tc.py -q -m gpu -x > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
for cfg in c2_image_512 c2_image_4096; do
  timeout 600 python bench.py --config $cfg --no-e2e > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err; echo "bench $cfg rc=$?"
done
timeout 600 python bench.py --config c3_blobs_1m_d64 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_c3.json 2>&1; echo "c3 rc=$?"
timeout 600 python bench.py --config c4_blobs_1m_large --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_c4.json 2>&1; echo "c4 rc=$?"
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/${tag}_bench_seed.json 2>&1; echo "seed rc=$?"
timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_c5.json 2>&1; echo "c5 rc=$?"
