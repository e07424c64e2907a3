# round 2, batch ax: segmented-gather flush variants (A: predicated RED per word, B: select chain, p2: shuffle wide path)
set -x
mkdir -p gpurun_out/ax
for C in 71429 15000; do
  for v in seg_A seg_B seg_p2; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1_seg,fused_seg,score2_seg,score4_seg,fused4_seg --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/ax/${v}_$C.log 2>&1; echo "$v $C"; cat gpurun_out/ax/${v}_$C.log
  done
done
