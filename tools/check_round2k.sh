#!/bin/bash
set -u
tag=${1:-round2k}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_c5_scale.py -q -m gpu -x > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 fp16', round(d['roofline']['avg_launch_ms'],4), 'ms', d['clocks']['sm_mhz'], d['value'])"
done
timeout 300 python bench.py --dist bf16 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 bf16', round(d['roofline']['avg_launch_ms'],4), 'ms', d['clocks']['sm_mhz'])"
timeout 300 python bench.py --config c3_blobs_1m_d64 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c3', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
