#!/bin/bash
set -u
run() { for cfg in c2_image_512 c2_image_4096 c1_blobs_small; do
  timeout 300 python bench.py --config $cfg --steps 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $cfg', round(d['roofline']['avg_launch_ms']*1e3,2), 'us')"; done; }
run default
MPK_NO_GRAPH=1 ncu --set full --clock-control none -k regex:smalld_iter --launch-skip 20 -c 1 -o gpurun_out/round2o_smalld_512 timeout 300 python bench.py --config c2_image_512 --steps 2 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
MPK_NVCC_EXTRA="-DMPK_SL_TILE=1024" python paper_2407_12208_b200/_build.py --force > /dev/null 2>&1; run tile1024
MPK_NVCC_EXTRA="-DMPK_SL_TILE=1024 -DMPK_SL_MINB=2" python paper_2407_12208_b200/_build.py --force > /dev/null 2>&1; run tile1024minb2
