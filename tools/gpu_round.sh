# full GPU pass: tests, smoke, bench (both arms), ncu launch list + full capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 300 python -m paper_2112_10034_b200 bench --iters 500 --repeats 5 > gpurun_out/cli_bench.txt 2>&1; echo clibench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'reduce_kernel|tile_tmem|hist256' -c 10 -f -o gpurun_out/kernels_full python tools/profile_kernels.py > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
python tools/launch_summary.py gpurun_out/launches.csv gpurun_out/launches_summary.md "launch list (ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 3 --warmup 3 --no-cpu-baseline)" > /dev/null; echo summary=$?
tail -3 gpurun_out/pytest_gpu.log; head -c 400 gpurun_out/bench.json
