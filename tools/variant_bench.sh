#!/bin/bash
# time the C5 distance kernel for the in-tree library and for prebuilt variants under
# tools/variants/*.so (swapped in place, restored at the end)
L=paper_2407_12208_b200/libmpkmeans.so
cp $L /tmp/lib_base.so
for v in /tmp/lib_base.so tools/variants/*.so; do
  cp $v $L
  for dist in ${DISTS:-fp16}; do
    timeout 300 python bench.py --steps 3 --warmup 3 --iters 10 --dist $dist --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$(basename $v)', '$dist', round(d['roofline']['avg_launch_ms'],3), 'ms', d['clocks'])"
  done
done
cp /tmp/lib_base.so $L
