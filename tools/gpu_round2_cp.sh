# round 2, batch cp: guarded tail batches of 6 / 8 vectors (one round trip for a short piece's rest) vs 4
set -x
mkdir -p gpurun_out/cp
for v in prod gt6 gt8; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 150 600 1500; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks $lib > gpurun_out/cp/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cp/${v}_$C.log
  done
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks $lib > gpurun_out/cp/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/cp/${v}_1m.log
done
