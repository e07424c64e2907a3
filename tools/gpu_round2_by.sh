# round 2, batch by: per-piece cost of the fused count-contract step: C = 1 / 50 / 150 / 300 chunks, product vs single worker (+stagger)
set -x
mkdir -p gpurun_out/by
for v in prod single single_st6; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 1 50 150 300; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4 $lib > gpurun_out/by/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/by/${v}_$C.log
  done
done
