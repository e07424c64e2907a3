# round 2, batch cc: the staggered single worker for the plain histogram, with piece caps of 1 / 2 / 4 MB
set -x
mkdir -p gpurun_out/cc
for v in prod hst hst_cap1m hst_cap2m hst_cap4m; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 1 150; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only hist,fused,score8 $lib > gpurun_out/cc/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cc/${v}_$C.log
  done
done
