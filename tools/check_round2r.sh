#!/bin/bash
set -u
timeout 900 python -m pytest tests/test_gpu_seed.py tests/test_gpu_image_sweep.py -q -m gpu > gpurun_out/round2r_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/round2r_tests.log
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/round2r_bench_seed.json 2>&1; echo "seed rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/round2r_bench_seed.json').read().strip().splitlines()[-1]); print('seed', d['value'], d['roofline']['frac'])"
timeout 600 python bench.py --seed-d2 --dist e5m2 --steps 2 > gpurun_out/round2r_bench_seed_e5m2.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/round2r_bench_seed_e5m2.json').read().strip().splitlines()[-1]); print('seed e5m2', d['value'], d['roofline']['frac'])"
