# round 2, batch u: CTA-pair (cta_group::2) contraction
set -x
mkdir -p gpurun_out/u
timeout 300 python -m pytest tests/test_gpu_contract.py -x -q -p no:cacheprovider > gpurun_out/u/tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -15 gpurun_out/u/tests.log
[ $rc -ne 0 ] && exit 1
timeout 300 python tools/probe_contract.py > gpurun_out/u/probe.json 2>&1; echo "probe rc=$?"
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_tc1.so timeout 300 python tools/probe_contract.py > gpurun_out/u/probe_tc1.json 2>&1; echo "probe1 rc=$?"
timeout 900 python bench.py --workload 4 --no-e2e > gpurun_out/u/bench_wl4.json 2> gpurun_out/u/bench_wl4.err; echo "bench4 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"contract_tc" -s 2 -c 2 -o gpurun_out/u/prof_tc2 python tools/prof_contract.py > gpurun_out/u/ncu.log 2>&1; echo "ncu rc=$?"
