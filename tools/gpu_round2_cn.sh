# round 2, batch cn: stagger the single worker in 4 / 8 groups of warps instead of 2 halves
set -x
mkdir -p gpurun_out/cn
for v in prod g4 g8; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 50 150 200; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,score8 $lib > gpurun_out/cn/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cn/${v}_$C.log
  done
done
