#!/bin/bash
# prep_vecg_kernel (d = 32 / 64): tests, C3 / C4 lines with and without
timeout 900 python -m pytest tests/test_gpu_prep_small.py tests/test_gpu_parity.py tests/test_gpu_virtual_ranks.py tests/test_gpu_tc.py -x -q --timeout 120 -k "not c5_shape" 2>&1 | tail -2
for v in "" 1; do
  export MPK_PREP_NO_VECG=$v; [ -z "$v" ] && unset MPK_PREP_NO_VECG
  for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
    set -- $cfg
    timeout 300 python bench.py --config $1 --dist $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('novecg=${v:-0} $1', '%.4g' % d['value'], d['unit'], round(d['ms_per_step'],4), 'ms/step prep', round(d['breakdown_ms_per_step']['prep'],3))"
  done
done
