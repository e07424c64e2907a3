# round 2, batch cq: final validation of the build - GPU suite, smoke, bench lines (configs 2/3/4/5, 140 tokens/chunk), reference arm
set -x
mkdir -p gpurun_out/cq
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/cq/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/cq/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/cq/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/cq/smoke.log
timeout 900 python bench.py > gpurun_out/cq/bench.json 2> gpurun_out/cq/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload 3 > gpurun_out/cq/bench_wl3.json 2> gpurun_out/cq/bench_wl3.err; echo "wl3 rc=$?"
timeout 900 python bench.py --workload 4 > gpurun_out/cq/bench_wl4.json 2> gpurun_out/cq/bench_wl4.err; echo "wl4 rc=$?"
timeout 900 python bench.py --workload 5 --no-cpu > gpurun_out/cq/bench_wl5.json 2> gpurun_out/cq/bench_wl5.err; echo "wl5 rc=$?"
timeout 900 python bench.py --chunks 71429 --no-cpu > gpurun_out/cq/bench_c71429.json 2> gpurun_out/cq/bench_c71429.err; echo "c71k rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/cq/ref.json 2> gpurun_out/cq/ref.err; echo "ref rc=$?"
