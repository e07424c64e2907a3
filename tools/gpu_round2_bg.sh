# round 2, batch bg: plain histogram on one 1024-thread worker (product) - GPU suite + kernel table
set -x
mkdir -p gpurun_out/bg
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bg/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bg/pytest.log
timeout 600 python tools/time_kernels.py --reps 10 --only hist,fused,score1,score4,hist_chunks > gpurun_out/bg/k150.log 2>&1; cat gpurun_out/bg/k150.log
timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only hist > gpurun_out/bg/k1500.log 2>&1; cat gpurun_out/bg/k1500.log
