#!/bin/bash
set -u
for dbg in 0 27; do
  MPK_PAIR_DBG=$dbg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:assign_pair --csv --log-file gpurun_out/round2s_dbg$dbg.csv python tools/pair_fixed_cost.py > /dev/null 2>&1
  echo "dbg $dbg rc=$?"
done
