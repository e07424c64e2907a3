# round 2, batch cj: staggered halves also inside the two 512-thread workers (pieces < 400 KB)
set -x
mkdir -p gpurun_out/cj
for v in prod st2_1000 st2_2000 st2_4000; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 300 600 1500; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks $lib > gpurun_out/cj/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cj/${v}_$C.log
  done
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks $lib > gpurun_out/cj/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/cj/${v}_1m.log
done
