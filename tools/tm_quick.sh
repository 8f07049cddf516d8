timeout 300 python -m pytest tests -x -q -m gpu -k "scan or compact" 2>&1 | tail -2
WF_SCAN_TMEM=1 timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | grep -v correct | sed "s/^/default /"
for lib in build/variants/lib_*.so; do case $lib in *trace*) continue;; esac; WF_LIB=$lib timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | sed "s#^#$(basename $lib) #"; done
for lib in build/variants/lib_*.so; do case $lib in *trace*) continue;; esac; WF_LIB=$lib timeout 300 python -m pytest tests -x -q -m gpu -k "scan or compact" 2>&1 | tail -1 | sed "s#^#$(basename $lib) #"; done
