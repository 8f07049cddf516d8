timeout 300 python -m pytest tests -x -q -m gpu -k "scan or compact" 2>&1 | tail -3
for v in 1 0; do WF_SCAN_TMEM=$v timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | sed "s/^/tmem=$v /"; done
for lib in build/variants/lib_*.so; do WF_LIB=$lib timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | sed "s#^#$(basename $lib) #"; done
