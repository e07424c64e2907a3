# round 2, batch bt: segmented gather W = 1 with 6 / 8 windows in flight per warp (1024-thread CTAs, redux flush) vs 4
set -x
mkdir -p gpurun_out/bt
for v in prod u6 u8; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 71429 15000 300; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1_seg,fused_seg $lib > gpurun_out/bt/${v}_$C.log 2>&1; echo "$v $C"; cat gpurun_out/bt/${v}_$C.log
  done
done
