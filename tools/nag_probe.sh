for v in nag2l3 nag2l6 nag2l4; do
  L=build/variants/lib_$v.so
  WF_LIB=$L timeout 200 python -m pytest tests -x -q -m gpu -k "scan or compact or tmem or misaligned" 2>&1 | tail -1 | sed "s/^/$v /"
  WF_LIB=$L timeout 100 python tools/stress_tmem.py 500 | sed "s/^/$v /"
  WF_LIB=$L timeout 100 python tools/bench_kernels.py c3 c4 | grep -v correct | sed "s/^/$v /"
done
timeout 100 python tools/bench_kernels.py c3 c4 | grep -v correct | sed "s/^/default /"
