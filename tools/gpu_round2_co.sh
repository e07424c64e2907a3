# round 2, batch co: the 1024-thread worker's flush spread over both halves (4 threads per bin) vs the lower half only
set -x
mkdir -p gpurun_out/co
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/co/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/co/tests.log
for v in prod tpb2; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 1 50 150 200; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,score8,hist_chunks $lib > gpurun_out/co/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/co/${v}_$C.log
  done
  timeout 600 python tools/time_kernels.py --reps 10 --only hist $lib > gpurun_out/co/${v}_hist.log 2>&1; cat gpurun_out/co/${v}_hist.log
done
