#!/bin/bash
# Launch list of the update kernels for a 2-iteration C5 fit: tools/upd_prof.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 python tools/one_fit.py 2 > gpurun_out/of.log 2>&1 || exit 1
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"block_|scan_|scatter|segsum|finalize|count_" --csv --log-file gpurun_out/upd.csv \
  python tools/one_fit.py 2 > /dev/null 2>&1
tail -1 gpurun_out/of.log
