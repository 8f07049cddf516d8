bash tools/red_sweep.sh
for v in build/variants/lib_*.so; do WF_LIB=$v bash tools/red_sweep.sh | grep "tma 1"; done
