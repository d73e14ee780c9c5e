#!/bin/bash
set -u
tag=${1:-round2i}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image_sweep.py tests/test_gpu_seed.py tests/test_gpu_virtual_ranks.py -q -m gpu > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/${tag}_bench_seed.json 2>&1; echo "seed rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/${tag}_bench_seed.json').read().strip().splitlines()[-1]); print('seed', d['value'], d['roofline']['frac'])"
for cfg in c2_image_512 c2_image_4096 c1_blobs_small; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench_${cfg}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/${tag}_bench_${cfg}.json').read().strip().splitlines()[-1]); print('$cfg', round(d['roofline']['avg_launch_ms']*1e3,2), 'us', d['roofline']['frac'])"
done
