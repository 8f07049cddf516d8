# compaction output-path variants (build with tools/build_variants.py first)
mkdir -p gpurun_out
python tools/bench_kernels.py ref > gpurun_out/sweep_compact.log 2>&1
for lib in build/variants/*.so; do echo "== $lib"; WF_LIB=$lib timeout 120 python tools/bench_kernels.py c3 c4; done >> gpurun_out/sweep_compact.log 2>&1
cat gpurun_out/sweep_compact.log
