# round 2, batch e: register-resident chunk bounds (segmented gather, dedup) + IMAD-balanced dedup record
set -x
mkdir -p gpurun_out/e
timeout 900 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/e/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/e/tests.log
ONLY=fused,score1,score2,score4,fused2,fused4,score1_seg,dedup
for C in 71429 15000 150; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only $ONLY > gpurun_out/e/new_$C.log 2>&1; echo "new $C rc=$?"
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only $ONLY --lib paper_2508_09229_b200/lib/libexp_old.so > gpurun_out/e/old_$C.log 2>&1; echo "old $C rc=$?"
done
