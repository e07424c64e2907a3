set -x
timeout 300 python -m pytest tests/test_gpu_contract.py -x -q -p no:cacheprovider > gpurun_out/contract_tests.log 2>&1; rc=$?; echo "contract tests rc=$rc"; tail -30 gpurun_out/contract_tests.log
[ $rc -ne 0 ] && exit 1
timeout 300 python tools/probe_contract.py > gpurun_out/probe_contract.json 2> gpurun_out/probe_contract.err; echo "probe rc=$?"
cat gpurun_out/probe_contract.json
timeout 600 python bench.py --workload 4 > gpurun_out/bench_wl4.json 2> gpurun_out/bench_wl4.err; echo "bench4 rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest.log
