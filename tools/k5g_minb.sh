#!/bin/bash
# K5g / K5p timings (4096^2 and 512^2 images, K5g forced for the latter) and the K5p/K5g tests
t() { timeout 300 python bench.py --config $1 --dist fp16 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$2 $1', round(d['roofline']['avg_launch_ms']*1000,2), 'us/iter', round(d['roofline']['frac'],4))"; }
t c2_image_4096 ""; MPK_NO_PERSIST=1 t c2_image_512 "K5g"; t c2_image_512 "K5p"
timeout 600 python -m pytest tests/test_gpu_smalld_persist.py tests/test_gpu_parity.py tests/test_gpu_image_sweep.py -q -x 2>&1 | tail -1
