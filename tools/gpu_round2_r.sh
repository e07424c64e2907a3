# round 2, batch r: one-hot server-mask dedup (<= 32 servers, costs <= 15) vs pairwise tests
set -x
mkdir -p gpurun_out/r
MP_STRESS_EXAMPLES=40 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_algos.py -x -q -p no:cacheprovider -k "dedup" > gpurun_out/r/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r/tests.log
for C in 150 15000 150000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only dedup > gpurun_out/r/onehot_$C.log 2>&1; echo "new $C rc=$?"
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only dedup --lib paper_2508_09229_b200/lib/libexp_pairwise.so > gpurun_out/r/pairwise_$C.log 2>&1; echo "old $C rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dedup_kernel" -c 1 -o gpurun_out/r/dedup150 python tools/prof_kernels.py --chunks 150 --which dedup --reps 1 > gpurun_out/r/ncu.log 2>&1; echo "ncu rc=$?"
