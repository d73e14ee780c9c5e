#!/bin/bash
# K5p without the stream synchronisation between the loop and the final pass: tests, C1/C2 lines
timeout 1200 python -m pytest tests/test_gpu_smalld_persist.py tests/test_gpu_prep_small.py tests/test_gpu_parity.py tests/test_gpu_image_sweep.py -x -q 2>&1 | tail -2
for cfg in c2_image_512 c1_blobs_small c2_image_4096; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$cfg', '%.4g' % d['value'], d['unit'], round(d['ms_per_step'],4), 'ms/step')"
done
