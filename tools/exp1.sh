set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "golden_fixtures or identical_fraction" 2>&1 | tail -2
for rep in 1 2; do
python tools/cfg_time.py --tag ffma
python tools/cfg_time.py --tag exact --exact
done
for h in 0 6 4 2 8 1; do
TAGG_L2_HINT=$h python tools/cfg_time.py ds_down ds_gateup q_fdn sweep_r64 --tag hint$h
done
for h in 0 6; do
TAGG_L2_HINT=$h ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tagg_gemm -s 3 -c 1 --csv python tools/cfg_time.py ds_down --iters 1 2>&1 | grep -E "dram__|gpu__time|hit_rate"
done
