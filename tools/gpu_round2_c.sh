timeout 300 python -m pytest tests/test_gpu_contract.py -x -q -p no:cacheprovider > gpurun_out/contract_tests.log 2>&1; rc=$?; echo "contract tests rc=$rc"; tail -15 gpurun_out/contract_tests.log
[ $rc -ne 0 ] && exit 1
timeout 300 python tools/probe_contract.py > gpurun_out/probe_v0.json 2>&1; echo "v0 rc=$?"
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_noatom.so timeout 300 python tools/probe_contract.py > gpurun_out/probe_noatom.json 2>&1; echo "noatom rc=$?"
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_nomma.so timeout 300 python tools/probe_contract.py > gpurun_out/probe_nomma.json 2>&1; echo "nomma rc=$?"
timeout 120 python tools/prof_contract.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"contract_tc|count_digits" -s 2 -c 2 -o gpurun_out/prof_contract2 python tools/prof_contract.py > gpurun_out/ncu_contract.log 2>&1; echo "ncu rc=$?"
