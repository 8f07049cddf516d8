mkdir -p gpurun_out
for lib in build/variants/*.so; do echo "== $lib"; WF_LIB=$lib WF_SCAN_PERSISTENT=1 timeout 120 python tools/bench_kernels.py c3 c4; done > gpurun_out/sweep3.log 2>&1
cat gpurun_out/sweep3.log
