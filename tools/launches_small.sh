#!/bin/bash
# ncu launch lists (kernel durations) of the C3 and C4 bench steps
mkdir -p gpurun_out
for cfg in "c4_blobs_1m_large e5m2" "c3_blobs_1m_d64 fp16"; do
  set -- $cfg
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv \
      timeout 600 python bench.py --config $1 --dist $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "$1 rc=$?"
  python tools/launch_summary.py gpurun_out/launches_$1.csv | head -24
done
