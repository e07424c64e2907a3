# round 2, batch bj: count-contract table words in registers again for W <= 4 (W = 8 reads them at the flush)
set -x
mkdir -p gpurun_out/bj
timeout 1200 python -m pytest tests/test_gpu_algos.py -x -q -p no:cacheprovider > gpurun_out/bj/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/bj/tests.log
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,score8,fused8 > gpurun_out/bj/k150.log 2>&1; cat gpurun_out/bj/k150.log
timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only fused,score4,score8 > gpurun_out/bj/k1500.log 2>&1; cat gpurun_out/bj/k1500.log
