for lib in build/variants/lib_*.so; do WF_LIB=$lib timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | grep us_median | sed "s#^#$(basename $lib) #"; done
