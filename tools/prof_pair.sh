set -u
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:"k<4>|_Z1kILi4" -c 1 -o gpurun_out/p_fold4 ./tools/fold_bench > gpurun_out/p_fold4.log 2>&1; echo "fold ncu rc=$?"
timeout 300 python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:assign_pair_kernel --launch-skip 4 -c 1 \
      -o gpurun_out/p_pair_full timeout 900 python bench.py --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e \
      > gpurun_out/p_ncu_full.log 2>&1
echo "pair ncu rc=$?"
