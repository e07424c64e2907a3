# round 2, batch aw: redux.sync flush in the segmented gather and dedup (product build) - parity + timing
set -x
mkdir -p gpurun_out/aw
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/aw/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/aw/tests.log
for C in 71429 15000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1_seg,fused_seg,score2_seg,score4_seg,fused4_seg > gpurun_out/aw/seg_$C.log 2>&1; cat gpurun_out/aw/seg_$C.log
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1_seg,fused_seg,score4_seg,fused4_seg --lib paper_2508_09229_b200/lib/libexp_seg_p2.so > gpurun_out/aw/seg_p2_$C.log 2>&1; cat gpurun_out/aw/seg_p2_$C.log
done
for C in 150 15000 150000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only dedup > gpurun_out/aw/dedup_$C.log 2>&1; cat gpurun_out/aw/dedup_$C.log
done
