mkdir -p gpurun_out
for lib in build/variants/lib_[!t]*.so; do echo "== $lib"; WF_LIB=$lib timeout 120 python tools/bench_kernels.py c3 c4; done > gpurun_out/sweep_tile.log 2>&1
for op in scan compact; do
for v in ${TRACES:-tra2}; do
WF_TRACE_OP=$op WF_TRACE_TILE=8192 WF_LIB=build/variants/lib_$v.so timeout 60 python tools/trace_scan.py >> gpurun_out/sweep_tile.log 2>&1
done
done
cat gpurun_out/sweep_tile.log
