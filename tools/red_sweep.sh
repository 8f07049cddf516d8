for v in default build/variants/lib_u2.so build/variants/lib_u8.so build/variants/lib_u16.so; do
  if [ $v = default ]; then L=""; else L="WF_LIB=$v"; fi
  env $L timeout 120 python tools/bench_kernels.py c2 c1 2>&1 | sed "s#^#$(basename $v) #"
done
