mkdir -p gpurun_out
for lib in build/variants/*.so; do
  for P in ${PERSIST:-1 0}; do
    echo "== $lib persist=$P"
    WF_LIB=$lib WF_SCAN_PERSISTENT=$P timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | tail -4
  done
done > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
