# round 2, batch bz: piece-end bytes counted after the vectors (no dependent byte loads ahead of warp 0's vector
# loads): per-piece cost at C = 1 / 50 / 150 / 300 / 1500 and config 4, product + single worker
set -x
mkdir -p gpurun_out/bz
for v in prod single single_st6; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 1 50 150 300 1500; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4 $lib > gpurun_out/bz/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/bz/${v}_$C.log
  done
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks $lib > gpurun_out/bz/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/bz/${v}_1m.log
done
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/bz/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/bz/tests.log
