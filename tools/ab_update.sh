#!/bin/bash
# A/B of the per-iteration update time: the tree vs the csrc files in ab_old/
set -u
rm -rf /tmp/abold && cp -r . /tmp/abold && cp ab_old/* /tmp/abold/paper_2407_12208_b200/csrc/
(cd /tmp/abold && python __graft_entry__.py build > /tmp/abold_build.log 2>&1) || { echo "old build failed"; tail -5 /tmp/abold_build.log; }
t() { (cd $1 && timeout 300 python bench.py --config $2 --dist $3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e) \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; it=d['config']['lloyd_iters_per_step']; print('$4 $2 $3 update us/iter', round(b['update']/it*1000,1))"; }
for rep in 1 2; do
for cfg in "c5_vq_10m fp16" "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $cfg
  t . $1 $2 new; t /tmp/abold $1 $2 old
done
done
