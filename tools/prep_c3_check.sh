#!/bin/bash
# prep-side changes at C3 / C4 (combine with a warp per column, block-reduced column maxima):
# tests, bench lines, launch lists
timeout 900 python -m pytest tests/test_gpu_prep_small.py tests/test_gpu_parity.py tests/test_gpu_virtual_ranks.py tests/test_gpu_tc.py -x -q --timeout 120 -k "not c5_shape" 2>&1 | tail -2
for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2" "c2_image_512 fp16"; do
  set -- $cfg
  timeout 300 python bench.py --config $1 --dist $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
    | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1', '%.4g' % d['value'], d['unit'], round(d['ms_per_step'],4), 'ms/step', {k: round(v,3) for k,v in d['breakdown_ms_per_step'].items()})"
done
bash tools/launches_small.sh
