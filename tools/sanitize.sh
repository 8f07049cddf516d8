mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_kernels.py 2>&1 | tail -8
done > gpurun_out/sanitize.log 2>&1
cat gpurun_out/sanitize.log
