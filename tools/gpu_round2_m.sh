# round 2, batch m: pipe_kernel as 1024-thread CTAs with two halves interleaved in 256-byte rows
set -x
mkdir -p gpurun_out/m
timeout 900 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/m/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/m/tests.log
for C in 150 1500; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score2,score4,hist_chunks,fused2,fused4 > gpurun_out/m/new_$C.log 2>&1; echo "new $C rc=$?"
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score2,score4,hist_chunks,fused2,fused4 --lib paper_2508_09229_b200/lib/libexp_split0.so > gpurun_out/m/old_$C.log 2>&1; echo "old $C rc=$?"
done
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/m/bench.json 2> gpurun_out/m/bench.err; echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -c 1 -o gpurun_out/m/pipe150 python tools/prof_kernels.py --chunks 150 --which fused --reps 1 > gpurun_out/m/ncu.log 2>&1; echo "ncu rc=$?"
