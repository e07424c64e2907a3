# round 2, batch x: full GPU suite + smoke + default bench + reference arm on HEAD
set -x
mkdir -p gpurun_out/x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/x/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/x/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/x/bench.json 2> gpurun_out/x/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/x/ref.json 2> gpurun_out/x/ref.err; echo "ref rc=$?"
