for rep in 1 2 3; do
for v in k2 k1 k3; do WF_LIB=build/variants/lib_$v.so timeout 100 python tools/bench_kernels.py c4 2>&1 | grep -v correct | sed "s#^#$v #"; done
done
