#!/bin/bash
# The evidence of profile_round2_final.sh without the ncu captures (for changes outside the
# pair kernel): GPU tests, smoke, the C5 lines and the supplementary configs.
set -u
tag=${1:-round2z}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${tag}_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${tag}_bench_c5_fp16.json 2> gpurun_out/${tag}_bench_c5_fp16.err; echo "bench rc=$?"
timeout 900 python bench.py --dist e5m2 > gpurun_out/${tag}_bench_c5_e5m2.json 2> gpurun_out/${tag}_bench_c5_e5m2.err; echo "e5m2 rc=$?"
for cfg in c2_image_512 c2_image_4096 c3_blobs_1m_d64 c4_blobs_1m_large c1_blobs_small; do
  timeout 600 python bench.py --config $cfg --no-e2e > gpurun_out/${tag}_bench_${cfg}.json 2> gpurun_out/${tag}_bench_${cfg}.err; echo "$cfg rc=$?"
done
timeout 900 python tools/image_sweep.py gpurun_out/${tag}_image_sweep.json > gpurun_out/${tag}_image_sweep.log 2>&1; echo "sweep rc=$?"
