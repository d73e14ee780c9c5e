#!/bin/bash
# ncu --set full of the persistent small-d loop (K5p) at C2 (512 x 512, fp16)
mkdir -p gpurun_out
timeout 300 python bench.py --config c2_image_512 --dist fp16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:smalld_iter_kernel --launch-skip 2 -c 1 \
    -o gpurun_out/p_k5p timeout 600 python bench.py --config c2_image_512 --dist fp16 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_k5p.log 2>&1
echo "ncu rc=$?"
