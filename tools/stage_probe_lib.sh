# DRAM / time of the probe shapes for the libraries given: bash tools/stage_probe_lib.sh lib1 lib2 ...
for cfg in "256 262144 7168 2048 zipf" "256 262144 7168 2048 uniform" "256 262144 4096 2048 uniform"; do
  set -- $cfg
  for lib in "${LIBS[@]}"; do
    cp build/ab/$lib.so paper_2508_16584_b200/libtagg.so
    r=$(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:tagg_gemm -s 1 -c 1 python tools/stage_probe.py $1 $2 $3 $4 0 $5 2 2>&1 | grep -E "dram__bytes_read|duration" | awk '{print $NF}' | tr '\n' ' ')
    echo "$cfg $lib -> $r"
  done
done
