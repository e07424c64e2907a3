# round 2, batch i: AUTO crossovers with the new segmented gather (forced algorithms, R1 10M tokens)
set -x
mkdir -p gpurun_out/i
ONLY=fused_count,fused_seg,fused_token,score1_gather,score1_seg,score1_token,score2_count,score2_seg,score4_count,score4_seg,fused2_count,fused2_seg,fused4_count,fused4_seg
for C in 150000 71429 15000 8000 5000 3000 2000 1500; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 3 --only $ONLY > gpurun_out/i/forced_$C.log 2>&1; echo "C $C rc=$?"
done
