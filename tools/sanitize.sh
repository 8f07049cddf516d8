# compute-sanitizer over every hot-path kernel (tools/sanitize_kernels.py)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --print-limit 40 python tools/sanitize_kernels.py 2>&1 | grep -v "^=========     \(Host\|Saved\| *#\)" | tail -60
done > gpurun_out/sanitize.log 2>&1
grep -c "Error\|Warning\|hazard" gpurun_out/sanitize.log
