for rep in 1 2 3; do
for v in prefuse current oldform; do WF_LIB=build/variants/lib_$v.so timeout 100 python tools/bench_kernels.py c4 c3 2>&1 | sed "s#^#$v #"; done
done
