# round 2, batch j: dedup warp ranges restructured (interior windows, progressive pick loads, no spills)
set -x
mkdir -p gpurun_out/j
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider -k "dedup or unique" > gpurun_out/j/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/j/tests.log
for C in 150 15000 150000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only dedup > gpurun_out/j/new_$C.log 2>&1; echo "new $C rc=$?"
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only dedup --lib paper_2508_09229_b200/lib/libexp_old.so > gpurun_out/j/old_$C.log 2>&1; echo "old $C rc=$?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dedup_kernel" -c 1 -o gpurun_out/j/dedup150 python tools/prof_kernels.py --chunks 150 --which dedup --reps 1 > gpurun_out/j/ncu.log 2>&1; echo "ncu rc=$?"
