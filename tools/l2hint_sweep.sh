for rep in 1 2 3; do
for v in cur ef cs efcs; do WF_LIB=build/variants/lib_$v.so timeout 100 python tools/bench_kernels.py c3 c4 2>&1 | sed "s#^#$v #"; done
done
