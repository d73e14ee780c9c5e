#!/bin/bash
python -m pytest tests/test_gpu_tc.py -x -q -k "one_tile or matches_oracle" 2>&1 | tail -1
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 $1 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"; }
for v in "" "-DMPK_PAIR_EARLY_REL=0"; do
  [ -n "$v" ] && MPK_NVCC_EXTRA="$v" python __graft_entry__.py build > /dev/null 2>&1
  t c3_blobs_1m_d64 fp16 "[$v]"; t c3_blobs_1m_d64 e5m2 "[$v]"; t c4_blobs_1m_large e5m2 "[$v]"; t c4_blobs_1m_large fp16 "[$v]"
done
