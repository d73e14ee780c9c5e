#!/bin/bash
# the d <= 4 row-per-thread kernels (prep, final assign, final SSE): bit-identity vs the general ones
# then C2 launch list (prep kernel time) with and without it
timeout 1200 python -m pytest tests/test_gpu_prep_small.py tests/test_gpu_parity.py tests/test_gpu_smalld_persist.py tests/test_gpu_image_sweep.py -x -q 2>&1 | tail -3
mkdir -p gpurun_out
t() { timeout 300 python bench.py --config $1 --dist $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 $1 $2', d['value'], d['unit'], round(d['ms_per_step'],4), 'ms/step')"; }
for v in "" 1; do
  export MPK_PREP_NO_SMALL=$v MPK_SIMT_NO_SMALL=$v; [ -z "$v" ] && unset MPK_PREP_NO_SMALL MPK_SIMT_NO_SMALL
  t c2_image_512 fp16 "nosmall=${v:-0}"; t c2_image_4096 fp16 "nosmall=${v:-0}"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prep_${v:-0}.csv \
      timeout 600 python bench.py --config c2_image_512 --dist fp16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_prep_${v:-0}.csv | head -12
done
