#!/bin/bash
# K5p (persistent small-d loop): parity vs K5g + oracle tests, then C1 / C2 timings with and
# without it
timeout 900 python -m pytest tests/test_gpu_smalld_persist.py tests/test_gpu_parity.py tests/test_gpu_image_sweep.py -x -q 2>&1 | tail -3
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 $1 $2', d['value'], d['unit'], round(d['ms_per_step'],4), 'ms/step', d.get('roofline',{}).get('frac'))"; }
for v in "" 1; do
  export MPK_NO_PERSIST=$v; [ -z "$v" ] && unset MPK_NO_PERSIST
  t c2_image_512 fp16 "persist=${v:-on}"; t c1_blobs_small fp64 "persist=${v:-on}"; t c2_image_4096 fp16 "persist=${v:-on}"
done
