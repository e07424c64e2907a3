# round 2, batch d: contraction with aligned split (tests, probe, config-4 bench + ncu launch list),
# config-3 (six topologies) bench, dialog-granularity timings (140 tokens per chunk)
set -x
mkdir -p gpurun_out/d
timeout 300 python -m pytest tests/test_gpu_contract.py -x -q -p no:cacheprovider > gpurun_out/d/contract_tests.log 2>&1; echo "contract tests rc=$?"; tail -3 gpurun_out/d/contract_tests.log
timeout 300 python tools/probe_contract.py > gpurun_out/d/probe_contract.json 2>&1; echo "probe rc=$?"
timeout 900 python bench.py --workload 4 > gpurun_out/d/bench_wl4.json 2> gpurun_out/d/bench_wl4.err; echo "bench4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d/launches_wl4.csv \
  python bench.py --workload 4 --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > gpurun_out/d/ncu_wl4.log 2>&1; echo "ncu4 rc=$?"
timeout 900 python bench.py --workload 3 > gpurun_out/d/bench_wl3.json 2> gpurun_out/d/bench_wl3.err; echo "bench3 rc=$?"
timeout 900 python tools/time_kernels.py --chunks 71429 --reps 5 --only fused,score1,score2,score4,fused2,fused4,fused_seg,fused_token,score4_seg,score4_token,hist > gpurun_out/d/tk_71429.log 2>&1; echo "tk rc=$?"
timeout 900 python tools/time_kernels.py --chunks 150 --reps 5 --only fused,score1,score4,fused_seg,hist,dedup > gpurun_out/d/tk_150.log 2>&1; echo "tk150 rc=$?"
