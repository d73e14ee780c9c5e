#!/bin/bash
set -u
timeout 300 python bench.py --seed-d2 --steps 1 --warmup 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seed --launch-skip 100 -c 40 --csv --log-file gpurun_out/round2q_seed_launches.csv timeout 600 python bench.py --seed-d2 --steps 1 --warmup 3 > /dev/null 2>&1
echo "rc=$?"
