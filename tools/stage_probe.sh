for cfg in "256 262144 7168 2048 zipf" "256 262144 7168 2048 uniform" "32 262144 7168 2048 uniform" "256 262144 4096 2048 uniform" "128 262144 4096 1536 uniform" "256 262144 7168 4096 uniform"; do
  set -- $cfg
  for f in 0 12288; do
    r=$(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:tagg_gemm -s 1 -c 1 python tools/stage_probe.py $1 $2 $3 $4 $f $5 2 2>&1 | grep -E "dram__bytes_read|duration" | awk '{print $NF}' | tr '\n' ' ')
    echo "$cfg flags=$f -> $r"
  done
done
