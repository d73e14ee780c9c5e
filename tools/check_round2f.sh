#!/bin/bash
set -u
tag=${1:-round2f}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_seed.py tests/test_gpu_image_sweep.py -q -m gpu > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --seed-d2 --steps 2 > gpurun_out/${tag}_bench_seed.json 2>&1; echo "seed rc=$?"
timeout 900 python bench.py --delta 2 --steps 2 --iters 5 --no-e2e > gpurun_out/${tag}_bench_delta2_c5.json 2>&1; echo "delta c5 rc=$?"
timeout 600 python bench.py --config c3_blobs_1m_d64 --delta 2 --steps 2 --iters 5 --no-e2e > gpurun_out/${tag}_bench_delta2_c3.json 2>&1; echo "delta c3 rc=$?"
MPK_MIXED_SIMT=1 timeout 600 python bench.py --config c3_blobs_1m_d64 --delta 2 --steps 2 --iters 5 --no-e2e > gpurun_out/${tag}_bench_delta2_c3_simt.json 2>&1; echo "delta c3 simt rc=$?"
for cfg in c2_image_512 c2_image_4096; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg default', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
done
MPK_NVCC_EXTRA="-DMPK_SL_MINB=2 -DMPK_SL_TILE=1024" python paper_2407_12208_b200/_build.py --force > gpurun_out/${tag}_rebuild.log 2>&1; echo "rebuild rc=$?"
for cfg in c2_image_512 c2_image_4096; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg minb2 tile1024', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"
done
