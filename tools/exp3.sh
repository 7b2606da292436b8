T="timeout 300"
for rep in 1 2; do
$T python tools/cfg_time.py --tag default
TAGG_STAGES=3 $T python tools/cfg_time.py --tag st3
TAGG_EPI_PASSES=2 $T python tools/cfg_time.py --tag epi2
TAGG_STAGES=4 $T python tools/cfg_time.py --tag st4
done
$T python tools/skinny_tiles.py
