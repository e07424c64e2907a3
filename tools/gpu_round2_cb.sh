# round 2, batch cb: why are 1.6 MB pieces (C = 50) faster than whole segments (C = 1)? piece cap 2 MB / 1 MB, per-CTA start stagger
set -x
mkdir -p gpurun_out/cb
for v in prod cap2m cap1m ctast; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 1 50 150; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only hist,fused $lib > gpurun_out/cb/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cb/${v}_$C.log
  done
done
