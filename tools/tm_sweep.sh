# timing of the default library and every variant in build/variants with
# tools/trace_tmem.py: scan + compaction at 0 / 50 % selectivity, 2^28 and 2^25;
# K2 (unchanged kernel) and nvidia-smi clocks as the box control
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw --format=csv
timeout 120 python tools/bench_kernels.py c2 2>&1 | grep '^{'
for lib in paper_2112_10034_b200/libwarpfold_b200.so build/variants/lib_*.so; do
  case $lib in *trace*) continue;; esac
  for lg in 28 25; do
    WF_LIB=$lib timeout 300 python tools/trace_tmem.py $lg 0 500 2>&1 | grep '^{'
  done
done
timeout 120 python tools/bench_kernels.py c2 2>&1 | grep '^{'
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw --format=csv
