timeout 100 python tools/bench_kernels.py c5 2>&1 | sed "s#^#default #"
for v in build/variants/lib_*.so; do WF_LIB=$v timeout 100 python tools/bench_kernels.py c5 2>&1 | sed "s#^#$(basename $v) #"; done
