#!/bin/bash
# ncu evidence for one round (run on the GPU box under gpurun): the headline launch list plus
# one full capture per kernel family.  Summaries: python tools/summarize_ncu.py <tag> <reps...>
set -u
mkdir -p gpurun_out
TAG=${1:-r01}
# 1. launch list of one bench step (127 GEMM launches): duration + DRAM bytes per launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:tagg_gemm -c 127 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --profile-once > gpurun_out/ncu_launches_${TAG}.log 2>&1
# 2. full captures: sweep launch r=64, DSv3 gate+up, DSv3 down, quantize+dispatch, wgrad
FULL="ncu --set full --clock-control none --import-source on"
$FULL -k regex:tagg_gemm -s 63 -c 1 -o gpurun_out/prof_${TAG} -f python bench.py --profile-once > gpurun_out/ncu_full_${TAG}.log 2>&1
$FULL -k regex:tagg_gemm -s 1 -c 1 -o gpurun_out/prof_ds_${TAG} -f python tools/prof_one.py ds_gateup 0 2 >> gpurun_out/ncu_full_${TAG}.log 2>&1
$FULL -k regex:tagg_gemm -s 1 -c 1 -o gpurun_out/prof_dsdown_${TAG} -f python tools/prof_one.py ds_down 0 2 >> gpurun_out/ncu_full_${TAG}.log 2>&1
$FULL -k regex:quantize_dispatch -s 1 -c 1 -o gpurun_out/prof_qd_${TAG} -f python tools/qd_bench.py >> gpurun_out/ncu_full_${TAG}.log 2>&1
$FULL -k regex:wgrad_kernel -s 1 -c 1 -o gpurun_out/prof_wg_${TAG} -f python tools/wg_bench.py >> gpurun_out/ncu_full_${TAG}.log 2>&1
# wg_bench launches per recipe: 2 warm-up + 5 timed each (per-column, 128x128 dY, MXFP8)
$FULL -k regex:wgrad_kernel -s 8 -c 1 -o gpurun_out/prof_wgb_${TAG} -f python tools/wg_bench.py >> gpurun_out/ncu_full_${TAG}.log 2>&1
$FULL -k regex:wgrad_kernel -s 15 -c 1 -o gpurun_out/prof_wgmx_${TAG} -f python tools/wg_bench.py >> gpurun_out/ncu_full_${TAG}.log 2>&1
# column-block quantizer, bf16 262144 x 2048: fp32-scale recipe, then MXFP8 (tools/colq_bench.py order)
$FULL -k regex:quantize_col_tile -s 2 -c 1 -o gpurun_out/prof_colq_${TAG} -f python tools/colq_bench.py >> gpurun_out/ncu_full_${TAG}.log 2>&1
$FULL -k regex:quantize_col_tile -s 9 -c 1 -o gpurun_out/prof_colqmx_${TAG} -f python tools/colq_bench.py >> gpurun_out/ncu_full_${TAG}.log 2>&1
echo "profile done"
