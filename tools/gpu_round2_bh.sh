# round 2, batch bh: 32-placement count-contract passes (W = 8): GPU suite, kernel timing, config 3 bench
set -x
mkdir -p gpurun_out/bh
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bh/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bh/pytest.log
timeout 600 python tools/time_kernels.py --reps 10 --only fused,score4,score8,fused4,fused8 > gpurun_out/bh/k150.log 2>&1; cat gpurun_out/bh/k150.log
timeout 900 python bench.py --workload 3 > gpurun_out/bh/bench_wl3.json 2> gpurun_out/bh/bench_wl3.err; echo "wl3 rc=$?"
timeout 900 python bench.py --workload 4 --no-cpu > gpurun_out/bh/bench_wl4.json 2> gpurun_out/bh/bench_wl4.err; echo "wl4 rc=$?"
timeout 900 python bench.py --no-cpu --sustained-s 0 > gpurun_out/bh/bench.json 2> gpurun_out/bh/bench.err; echo "wl2 rc=$?"
