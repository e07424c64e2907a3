# round 2, batch cl: the single staggered worker for every piece length (after the end-byte fix) vs the product
set -x
mkdir -p gpurun_out/cl
for v in prod allsingle; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 200 300 600 1500; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks $lib > gpurun_out/cl/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cl/${v}_$C.log
  done
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks $lib > gpurun_out/cl/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/cl/${v}_1m.log
done
