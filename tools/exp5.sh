mkdir -p gpurun_out/sanitizer_r02
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize.py > gpurun_out/sanitizer_r02/$t.txt 2>&1
  tail -3 gpurun_out/sanitizer_r02/$t.txt
done
timeout 300 python -m pytest tests/test_wgrad_gpu.py tests/test_moe_gpu.py -q -x 2>&1 | tail -3
TAGG_COLQ_V8=1 timeout 120 python tools/colq_bench.py
timeout 120 python tools/colq_bench.py
