# round 2, batch bn: explicit small carveout preference (0 %: max L1) for the streaming kernels vs the runtime default
set -x
mkdir -p gpurun_out/bn
for v in prod carve0 carve58; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist $lib > gpurun_out/bn/$v.log 2>&1; echo "$v"; cat gpurun_out/bn/$v.log
  timeout 600 python tools/time_kernels.py --chunks 71429 --reps 10 --only fused_seg,score1_seg,score4_seg $lib > gpurun_out/bn/${v}_71k.log 2>&1; cat gpurun_out/bn/${v}_71k.log
done
