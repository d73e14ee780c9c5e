#!/bin/bash
# one-tile grouped row-blocks: parity subset + C3 / C4 launch times vs MPK_PAIR_RBR, then the
# two-MMA-warp variant
python -m pytest tests/test_gpu_tc.py -x -q -k "one_tile or matches_oracle or final or ties or nonfinite" 2>&1 | tail -2
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 $1 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"; }
t c3_blobs_1m_d64 fp16 base
for R in 4 2 1; do
  MPK_PAIR_RBR=$R t c4_blobs_1m_large e5m2 R=$R
  MPK_PAIR_RBR=$R t c4_blobs_1m_large fp16 R=$R
done
MPK_NVCC_EXTRA="-DMPK_PAIR_MMA2=1" python __graft_entry__.py build > /dev/null 2>&1
t c3_blobs_1m_d64 fp16 mma2
t c4_blobs_1m_large e5m2 mma2
t c4_blobs_1m_large fp16 mma2
