# round 2, batch ae: next-chunk-bound prefetch in pipe_kernel
set -x
mkdir -p gpurun_out/ae
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/ae/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ae/tests.log
for C in 150 300 1500; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks > gpurun_out/ae/new_$C.log 2>&1
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks --lib paper_2508_09229_b200/lib/libexp_head.so > gpurun_out/ae/old_$C.log 2>&1
done
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks > gpurun_out/ae/new_1m.log 2>&1
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks --lib paper_2508_09229_b200/lib/libexp_head.so > gpurun_out/ae/old_1m.log 2>&1
