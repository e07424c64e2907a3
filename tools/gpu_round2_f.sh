# round 2, batch f: ncu --set full of the short-chunk kernels (SEG at 140 tokens/chunk) and dedup
set -x
mkdir -p gpurun_out/f
timeout 300 python tools/prof_kernels.py --chunks 71429 --which score1_seg,fused_seg,score4_seg,dedup --reps 1 > gpurun_out/f/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel|dedup_kernel" -c 4 -o gpurun_out/f/seg71k python tools/prof_kernels.py --chunks 71429 --which score1_seg,fused_seg,score4_seg,dedup --reps 1 > gpurun_out/f/ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel" -c 1 -o gpurun_out/f/seg150 python tools/prof_kernels.py --chunks 150 --which score1_seg --reps 1 > gpurun_out/f/ncu150.log 2>&1; echo "ncu150 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -c 1 -o gpurun_out/f/pipe150 python tools/prof_kernels.py --chunks 150 --which fused --reps 1 > gpurun_out/f/ncup.log 2>&1; echo "ncupipe rc=$?"
