# ROUND-1 RECORD: used runtime switches (WF_SCAN_2P / WF_SCAN_TMEM) that round 2
# removed from the product library; the round-1 kernels build only as variants
# (tools/build_variants.py with -DWF_SCAN_IMPL=1|2|3), selected with WF_LIB.
timeout 300 python -m pytest tests -x -q -m gpu -k "scan or compact or reference_pins or tmem" 2>&1 | tail -2
WF_SCAN_TMEM=1 timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | grep -v correct | sed "s/^/default /"
for lib in build/variants/lib_*.so; do case $lib in *trace*) continue;; esac; WF_LIB=$lib timeout 120 python tools/bench_kernels.py c3 c4 2>&1 | grep -v correct | sed "s#^#$(basename $lib) #"; done
[ -f build/variants/lib_trace.so ] && WF_LIB=build/variants/lib_trace.so timeout 300 python tools/trace_tmem.py
