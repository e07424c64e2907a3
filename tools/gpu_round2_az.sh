# round 2, batch az: segmented gather with one 1024-thread CTA per SM (tables + histogram below 96 KB) vs two 512-thread CTAs
set -x
mkdir -p gpurun_out/az
for C in 71429 15000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1_seg,fused_seg,score2_seg,fused2_seg,score4_seg,fused4_seg > gpurun_out/az/p_$C.log 2>&1; echo "product $C"; cat gpurun_out/az/p_$C.log
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1_seg,fused_seg,score2_seg,fused2_seg,score4_seg,fused4_seg --lib paper_2508_09229_b200/lib/libexp_seg1024.so > gpurun_out/az/t_$C.log 2>&1; echo "1024 $C"; cat gpurun_out/az/t_$C.log
done
