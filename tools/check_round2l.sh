#!/bin/bash
set -u
tag=${1:-round2l}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py -q -m gpu -x -k "assign_matches or deep or ties or nonfinite" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
run() { for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 c5 fp16', round(d['roofline']['avg_launch_ms'],4), 'ms', d['clocks']['sm_mhz'])"; done; }
run early
MPK_NVCC_EXTRA="-DMPK_PAIR_CNINIT_EARLY=0" python paper_2407_12208_b200/_build.py --force > /dev/null 2>&1; run late
MPK_NVCC_EXTRA="-DMPK_PAIR_CNINIT=0" python paper_2407_12208_b200/_build.py --force > /dev/null 2>&1; run off
