#!/bin/bash
set -u
tag=${1:-round2e}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_image_sweep.py tests/test_gpu_seed.py tests/test_gpu_parity.py -q -m gpu -k "pow2 or mx or seed or c1 or c2 or step" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/${tag}_bench_seed.json 2>&1; echo "seed rc=$?"
for cfg in c2_image_512 c2_image_4096; do
  MPK_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:smalld_iter --launch-skip 8 -c 1 \
    -o gpurun_out/${tag}_smalld_${cfg} timeout 600 python bench.py --config $cfg --steps 1 --warmup 3 --iters 4 \
    --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_smalld_${cfg}.log 2>&1
  echo "ncu smalld $cfg rc=$?"
done
ncu --set full --import-source on --clock-control none -k regex:seed_update --launch-skip 20 -c 1 \
    -o gpurun_out/${tag}_seed timeout 600 python bench.py --seed-d2 --steps 1 --warmup 3 > gpurun_out/${tag}_ncu_seed.log 2>&1
echo "ncu seed rc=$?"
