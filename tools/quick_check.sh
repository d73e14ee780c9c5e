#!/bin/bash
# Iteration loop on the GPU box: distance-kernel parity tests, then the C5 bench line (kernel
# time, roofline fraction, clocks). Usage: tools/quick_check.sh <tag> [pytest -k expr]
tag=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x ${2:+-k "$2"} > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
python - "$tag" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/{sys.argv[1]}_bench.json"))
r = d["roofline"]
print("value %.4g ms/step %.2f dist %.3f ms frac %.4f clocks %s" % (d["value"], d["ms_per_step"], r["avg_launch_ms"], r["frac"], d["clocks"]))
print(d.get("breakdown_ms_per_step"))
PY
