#!/bin/bash
set -u
tag=${1:-round2h}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image_sweep.py -q -m gpu > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
for cfg in c2_image_512 c2_image_4096 c1_blobs_small; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_${cfg}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/${tag}_bench_${cfg}.json').read().strip().splitlines()[-1]); print('$cfg', round(d['roofline']['avg_launch_ms']*1e3,2), 'us', d['roofline']['frac'])"
done
MPK_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:smalld_iter --launch-skip 8 -c 1 \
    -o gpurun_out/${tag}_smalld_4096 timeout 600 python bench.py --config c2_image_4096 --steps 1 --warmup 3 --iters 4 \
    --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_smalld.log 2>&1
echo "ncu smalld rc=$?"
ncu --set full --import-source on --clock-control none -k regex:seed_update --launch-skip 20 -c 1 \
    -o gpurun_out/${tag}_seed timeout 600 python bench.py --seed-d2 --steps 1 --warmup 3 > gpurun_out/${tag}_ncu_seed.log 2>&1
echo "ncu seed rc=$?"
