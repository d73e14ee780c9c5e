#!/bin/bash
# rbh (row-block halves): pair-kernel parity subset, then A/B of C5 / C3 launch times vs ab_old/
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_c5_scale.py -x -q 2>&1 | tail -2
bash tools/ab_pair.sh
t() { (cd $1 && timeout 300 python bench.py --config c3_blobs_1m_d64 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e) \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 c3 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"; }
t . fp16 new; t /tmp/abold fp16 old
for rep in 1 2; do (timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e) | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('new full-step', round(d['value']/1e12,3), 'e12 evals/s', round(d['roofline']['avg_launch_ms'],3), 'ms clk', d['clocks']['sm_mhz'])"; (cd /tmp/abold && timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e) | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('old full-step', round(d['value']/1e12,3), 'e12 evals/s', round(d['roofline']['avg_launch_ms'],3), 'ms clk', d['clocks']['sm_mhz'])"; done
