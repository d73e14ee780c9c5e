python -m pytest tests/test_gpu_tc.py -x -q -k "one_tile or deep_row or matches_oracle" 2>&1 | tail -5
for cfg in "c3_blobs_1m_d64 fp16" "c3_blobs_1m_d64 e5m2" "c4_blobs_1m_large e5m2" "c4_blobs_1m_large fp16"; do
  set -- $cfg
  for dbg in 0 32; do
    MPK_PAIR_DBG=$dbg timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $2 dbg=$dbg', round(d['roofline']['avg_launch_ms']*1000,1), 'us', d['value'])"
  done
done
