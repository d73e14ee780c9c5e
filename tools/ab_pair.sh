#!/bin/bash
# A/B of the pair kernel: the current tree vs the files in ab_old/ (built in a copy under /tmp),
# C5 fp16 / E5M2 launch times, interleaved runs
set -u
rm -rf /tmp/abold && cp -r . /tmp/abold && cp ab_old/* /tmp/abold/paper_2407_12208_b200/csrc/
(cd /tmp/abold && python __graft_entry__.py build > /tmp/abold_build.log 2>&1) || { echo "old build failed"; tail -5 /tmp/abold_build.log; }
t() { (cd $1 && timeout 300 python bench.py --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e) \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$3 $2', round(d['roofline']['avg_launch_ms']*1000,1), 'us clk', d['clocks']['sm_mhz'])"; }
for rep in 1 2; do
  for dist in fp16 e5m2; do t . $dist new; t /tmp/abold $dist old; done
done
