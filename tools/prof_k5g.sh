#!/bin/bash
# ncu --set full of K5g on the 4096^2 image (fp16)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:smalld_iter_kernel --launch-skip 3 -c 1 \
    -o gpurun_out/p_k5g timeout 600 python bench.py --config c2_image_4096 --dist fp16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/p_k5g.log 2>&1
echo "ncu rc=$?"
