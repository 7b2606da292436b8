#!/bin/bash
# tools/cyc_ab.sh A.so B.so ... -- shapes...   (on the GPU box; see tools/cyc_ab.py)
mkdir -p gpurun_out
ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/cyc.csv python tools/cyc_ab.py "$@" > /dev/null 2>&1
python tools/cyc_ab.py --report gpurun_out/cyc.csv "$@"
