# round 2, batch p: full GPU suite + smoke + default bench (+ ncu launch list) + reference arm on HEAD
set -x
mkdir -p gpurun_out/p
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/p/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/p/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/p/bench.json 2> gpurun_out/p/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/p/ref.json 2> gpurun_out/p/ref.err; echo "ref rc=$?"
timeout 900 python bench.py --chunks 71429 --no-cpu > gpurun_out/p/bench_c71429.json 2> gpurun_out/p/bench_c71429.err; echo "bench71k rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > gpurun_out/p/ncu.log 2>&1; echo "ncu rc=$?"
