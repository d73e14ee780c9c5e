#!/bin/bash
# one-tile parity tests + C3 / C4 launch times (default and MPK_PAIR_DBG extra settings)
python -m pytest tests/test_gpu_tc.py -x -q -k "one_tile" 2>&1 | tail -2
for cfg in "c3_blobs_1m_d64 fp16" "c3_blobs_1m_d64 e5m2" "c4_blobs_1m_large e5m2" "c4_blobs_1m_large fp16"; do
  set -- $cfg
  for env in "X=0" "$@"; do :; done
  timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"
done
