#!/bin/bash
# Round-2: pair-kernel traces at C3/C4, debug-mode split timings, smalld / seeding captures,
# compute-sanitizer memcheck of every kernel family.
set -u
tag=${1:-round2d}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1 or c2 or step" > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $cfg
  MPK_PAIR_TRACE=gpurun_out/${tag}_trace_$1.txt timeout 300 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  for dbg in 0 1 2 3; do
    MPK_PAIR_DBG=$dbg timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 dbg=$dbg', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
  done
done
MPK_NO_GRAPH=1 timeout 300 python bench.py --config c2_image_512 --steps 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c2 512 nograph', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
MPK_NO_FUSED_LOOP=1 timeout 300 python bench.py --config c2_image_512 --steps 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c2 512 unfused', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
MPK_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:smalld_iter --launch-skip 30 -c 1 \
    -o gpurun_out/${tag}_smalld_4096 timeout 600 python bench.py --config c2_image_4096 --steps 1 --warmup 3 --iters 4 \
    --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_smalld.log 2>&1
echo "ncu smalld rc=$?"
ncu --set full --import-source on --clock-control none -k regex:seed_update --launch-skip 20 -c 1 \
    -o gpurun_out/${tag}_seed timeout 600 python bench.py --seed-d2 --steps 1 --warmup 3 > gpurun_out/${tag}_ncu_seed.log 2>&1
echo "ncu seed rc=$?"
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/${tag}_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -3 gpurun_out/${tag}_memcheck.log
