#!/bin/bash
# Evidence for profiles/: bench line (both arms), ncu launch list of the bench command, one
# ncu --set full capture of the distance kernel. Each ncu pass runs only after the same command
# exited 0 without ncu. Usage: tools/profile_round.sh <tag>
set -u
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; rc=$?
echo "bench rc=$rc"
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
echo "reference rc=$?"
if [ $rc -eq 0 ]; then
  timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
      timeout 1200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu_launch.log 2>&1
  echo "launch list rc=$?"
  ncu --set full --import-source on --clock-control none -k regex:assign_pair_kernel --launch-skip 4 -c 1 \
      -o gpurun_out/${tag}_pair_full timeout 900 python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e \
      > gpurun_out/${tag}_ncu_full.log 2>&1
  echo "full capture rc=$?"
fi
