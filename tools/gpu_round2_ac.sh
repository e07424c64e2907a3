set -x
mkdir -p gpurun_out/ac
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_algos.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/ac/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ac/tests.log
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only hist,fused > gpurun_out/ac/t.log 2>&1; cat gpurun_out/ac/t.log
