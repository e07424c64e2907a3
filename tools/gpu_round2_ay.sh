# round 2, batch ay: AUTO crossovers re-measured after the redux.sync flush (forced algorithms, R1 10M)
set -x
mkdir -p gpurun_out/ay
for C in 150000 100000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only score1_seg,score1_token > gpurun_out/ay/c$C.log 2>&1; echo "C=$C"; cat gpurun_out/ay/c$C.log
done
for C in 1000 1500 2000 3333 5000; do
  timeout 900 python tools/time_kernels.py --chunks $C --reps 5 --only fused_seg,fused_count,score2_seg,score2_count,score4_seg,score4_count,fused2_seg,fused2_count,fused4_seg,fused4_count > gpurun_out/ay/c$C.log 2>&1; echo "C=$C"; cat gpurun_out/ay/c$C.log
done
for C in 300 500 700; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only score1_seg,score1_gather > gpurun_out/ay/s$C.log 2>&1; echo "C=$C"; cat gpurun_out/ay/s$C.log
done
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/ay/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ay/tests.log
