#!/bin/bash
# pair-kernel parity subset + launch times at C3 / C4 / C5
python -m pytest tests/test_gpu_tc.py -x -q -k "one_tile or deep_row or matches_oracle or final" 2>&1 | tail -2
for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2" "c5_vq_10m fp16" "c5_vq_10m e5m2"; do
  set -- $cfg
  timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters ${ITERS:-10} --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us', 'clk', d['clocks']['sm_mhz'])"
done
