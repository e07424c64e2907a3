# round 2, batch s: L2 prefetch past each piece in pipe_kernel (config-4 per-chunk histogram, 1M tokens)
set -x
mkdir -p gpurun_out/s
for v in base pf32768 pf65536 pf131072; do
  lib=""; [ $v != base ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 150 1500; do
    timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks $C --reps 20 --only hist_chunks,fused,score4 $lib > gpurun_out/s/${v}_1m_$C.log 2>&1
  done
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,hist_chunks,score4 $lib > gpurun_out/s/${v}_10m_150.log 2>&1
  timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only fused,hist_chunks,score4 $lib > gpurun_out/s/${v}_10m_1500.log 2>&1
  echo "$v done"
done
