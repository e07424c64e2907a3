# round 2, batch cs: validation of the final HEAD - GPU suite, smoke, default bench, config 4
set -x
mkdir -p gpurun_out/cs
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/cs/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/cs/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/cs/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/cs/bench.json 2> gpurun_out/cs/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload 4 > gpurun_out/cs/bench_wl4.json 2> gpurun_out/cs/bench_wl4.err; echo "wl4 rc=$?"
