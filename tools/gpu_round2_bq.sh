# round 2, batch bq: validation of the current build - GPU suite, smoke, bench lines (configs 2, 3, 4, 140 tokens/chunk), reference arm
set -x
mkdir -p gpurun_out/bq
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bq/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bq/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bq/smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/bq/smoke.log | tail -3
timeout 900 python bench.py > gpurun_out/bq/bench.json 2> gpurun_out/bq/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload 3 > gpurun_out/bq/bench_wl3.json 2> gpurun_out/bq/bench_wl3.err; echo "wl3 rc=$?"
timeout 900 python bench.py --workload 4 > gpurun_out/bq/bench_wl4.json 2> gpurun_out/bq/bench_wl4.err; echo "wl4 rc=$?"
timeout 900 python bench.py --chunks 71429 --no-cpu > gpurun_out/bq/bench_c71429.json 2> gpurun_out/bq/bench_c71429.err; echo "c71k rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bq/ref.json 2> gpurun_out/bq/ref.err; echo "ref rc=$?"
