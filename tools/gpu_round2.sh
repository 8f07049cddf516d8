# full GPU pass (round 2): smoke, -m gpu suite, bench (both arms), ncu launch
# list of the bench command and one --set full capture of every hot kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'reduce_kernel|tile_tmem|hist256|warp_partials|warp_prefix32' -c 14 -f -o gpurun_out/kernels_full python tools/profile_kernels.py > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
tail -3 gpurun_out/pytest_gpu.log; head -c 300 gpurun_out/bench.json
