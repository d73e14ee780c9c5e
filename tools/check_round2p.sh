#!/bin/bash
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_image_sweep.py -q -m gpu -k "c1 or c2 or image" > gpurun_out/round2p_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/round2p_tests.log
for cfg in c2_image_512 c2_image_4096 c1_blobs_small; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"; done
