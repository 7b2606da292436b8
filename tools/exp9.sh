for mode in 0 1 2; do for mb in 16 48; do
timeout 120 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum --clock-control none -k regex:stream_all --csv ./tools/micro/l2_dies $mode $mb 2>&1 | grep -E "mode|dram__bytes_read|lts__t_sectors" 
done; done
