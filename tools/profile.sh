#!/bin/bash
# ncu evidence for the headline workload (run on the GPU box under gpurun).
#  1. launch list of one bench step (127 GEMM launches): duration + DRAM bytes per launch
#  2. one full capture of a representative launch (r = 64, launch index 63)
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:tagg_gemm -c 127 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --profile-once > gpurun_out/ncu_launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tagg_gemm -s 63 -c 1 \
    -o gpurun_out/prof_${TAG} -f python bench.py --profile-once > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "profile done"
