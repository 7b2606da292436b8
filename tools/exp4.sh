bash tools/prof_skinny.sh
timeout 120 compute-sanitizer --tool racecheck ./tools/micro/alloc_race 2 > gpurun_out/alloc_race_cg2.txt 2>&1
timeout 120 compute-sanitizer --tool racecheck ./tools/micro/alloc_race 1 > gpurun_out/alloc_race_cg1.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
tail -2 gpurun_out/r2_bench4.err
cat gpurun_out/alloc_race_cg2.txt gpurun_out/alloc_race_cg1.txt
