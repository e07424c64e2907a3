# round 2, batch h: segmented gather with compile-time interior windows, 32-bit bound reloads
set -x
mkdir -p gpurun_out/h
timeout 900 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/h/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/h/tests.log
ONLY=fused_seg,score1_seg,score2_seg,score4_seg,fused2_seg,fused4_seg,fused,score1,score4
for C in 71429 15000 150; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only $ONLY > gpurun_out/h/new_$C.log 2>&1; echo "new $C rc=$?"
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only $ONLY --lib paper_2508_09229_b200/lib/libexp_old.so > gpurun_out/h/old_$C.log 2>&1; echo "old $C rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_kernel" -c 3 -o gpurun_out/h/seg71k python tools/prof_kernels.py --chunks 71429 --which score1_seg,fused_seg,score4_seg --reps 1 > gpurun_out/h/ncu.log 2>&1; echo "ncu rc=$?"
