# ncu per-launch DRAM bytes and duration of the skinny launches (tools/prof_skinny.py)
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for r in 1 8 64; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm|pad" -s 2 --csv python tools/prof_skinny.py free $r > gpurun_out/ncu_skinny_free_r$r.csv 2>&1
done
for r in 1 64; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm|pad" -s 6 --csv python tools/prof_skinny.py padded $r > gpurun_out/ncu_skinny_padded_r$r.csv 2>&1
done
timeout 300 ncu --metrics $M --clock-control none -k regex:"pad_groups|unpad_rows" -s 4 --csv python tools/prof_skinny.py padbig 0 > gpurun_out/ncu_padbig.csv 2>&1
