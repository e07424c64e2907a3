# round 2, batch ar: bench (config 2, default; config 3; config 4; 140 tokens/chunk) + GPU suite + smoke + ncu launch list
set -x
mkdir -p gpurun_out/ar
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ar/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ar/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ar/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/ar/bench.json 2> gpurun_out/ar/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload 3 > gpurun_out/ar/bench_wl3.json 2> gpurun_out/ar/bench_wl3.err; echo "bench3 rc=$?"
timeout 900 python bench.py --workload 4 > gpurun_out/ar/bench_wl4.json 2> gpurun_out/ar/bench_wl4.err; echo "bench4 rc=$?"
timeout 900 python bench.py --chunks 71429 --no-cpu > gpurun_out/ar/bench_c71429.json 2> gpurun_out/ar/bench_c71429.err; echo "bench71k rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ar/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > gpurun_out/ar/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -c 1 -o gpurun_out/ar/pipe150 python tools/prof_kernels.py --chunks 150 --which fused --reps 1 > gpurun_out/ar/ncu_full.log 2>&1; echo "ncu full rc=$?"
