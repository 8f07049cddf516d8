for rep in 1 2; do
for v in d16 d1a d1b d1c d2b d16b; do WF_LIB=build/variants/lib_$v.so timeout 100 python tools/bench_kernels.py c3 c4 2>&1 | grep -v correct | sed "s#^#$v #"; done
done
