#!/bin/bash
# Compile-time variants of the pair kernel at C3 (fp16), C4 (E5M2) and C5 (fp16, E5M2):
# spinning vs suspending waits of the role warps, 4 epilogue warpgroups.
set -u
run() {
  for spec in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2" "c5_vq_10m fp16" "c5_vq_10m e5m2"; do
    set -- $spec
    timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$VAR', '$1', '$2', round(d['roofline']['avg_launch_ms']*1e3,2), 'us', d['clocks']['sm_mhz'])"
  done
}
VAR=default; run
for v in "-DMPK_PAIR_HOT_RING=0" "-DMPK_PAIR_HOT_RING=0 -DMPK_PAIR_HOT_WAIT=0" "-DMPK_PAIR_EWG=4"; do
  MPK_NVCC_EXTRA="$v" python paper_2407_12208_b200/_build.py --force > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  VAR="$v"; run
done
