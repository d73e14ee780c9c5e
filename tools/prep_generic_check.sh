#!/bin/bash
# launch_prep through the lane-group / float4 kernels for large fp32 row sets: all GPU tests,
# smoke, the E5M2 C5 and C4 lines with and without (MPK_PREP_GENERIC=1)
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 300 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1; echo "smoke rc=$?"
for v in "" 1; do
  export MPK_PREP_GENERIC=$v; [ -z "$v" ] && unset MPK_PREP_GENERIC
  for cfg in "c5_vq_10m e5m2" "c4_blobs_1m_large e5m2"; do
    set -- $cfg
    timeout 600 python bench.py --config $1 --dist $2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('generic=${v:-0} $1', '%.4g' % d['value'], round(d['ms_per_step'],3), 'ms/step final', round(d['breakdown_ms_per_step']['final'],3))"
  done
done
