# round 2, batch ad: run streaming across piece boundaries in pipe_kernel
set -x
mkdir -p gpurun_out/ad
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/ad/tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/ad/tests.log
[ $rc -ne 0 ] && exit 1
for C in 1 50 150 300 1500; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score2,score4,hist_chunks > gpurun_out/ad/new_$C.log 2>&1
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score2,score4,hist_chunks --lib paper_2508_09229_b200/lib/libexp_noruns.so > gpurun_out/ad/old_$C.log 2>&1
  echo "C=$C done"
done
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks > gpurun_out/ad/new_1m.log 2>&1
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks --lib paper_2508_09229_b200/lib/libexp_noruns.so > gpurun_out/ad/old_1m.log 2>&1
