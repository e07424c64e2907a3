# round 2, batch ba: full GPU suite + smoke + bench lines (default, 140 tokens/chunk) after the SEG changes
set -x
mkdir -p gpurun_out/ba
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ba/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ba/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ba/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/ba/bench.json 2> gpurun_out/ba/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --chunks 71429 --no-cpu > gpurun_out/ba/bench_c71429.json 2> gpurun_out/ba/bench_c71429.err; echo "bench71k rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel" -c 3 -o gpurun_out/ba/seg71k python tools/prof_kernels.py --chunks 71429 --which score1_seg,fused_seg,score4_seg --reps 1 > gpurun_out/ba/ncu_seg.log 2>&1; echo "ncu rc=$?"
