#!/bin/bash
# C3 / C4 launch time vs the X~ ring depth (MPK_PAIR_SA) and accumulator count (MPK_PAIR_NACC),
# plus a clock64 trace of the default configuration
mkdir -p gpurun_out
for cfg in "c3_blobs_1m_d64 fp16" "c4_blobs_1m_large e5m2"; do
  set -- $cfg
  MPK_PAIR_TRACE=gpurun_out/trace_rbalt_${1}.txt timeout 300 python bench.py --config $1 --dist $2 --steps 1 --warmup 3 --iters 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  for v in "4 4" "8 4" "4 8" "8 8" "16 8"; do
    set -- $cfg $v
    MPK_PAIR_SA=$3 MPK_PAIR_NACC=$4 timeout 300 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --iters 10 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1 $2 SA=$3 NACC=$4', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"
  done
done
