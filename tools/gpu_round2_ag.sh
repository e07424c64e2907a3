set -x
mkdir -p gpurun_out/ag
for C in 1 150; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -c 1 -o gpurun_out/ag/pipe_c$C python tools/prof_kernels.py --chunks $C --which fused --reps 1 > gpurun_out/ag/ncu_c$C.log 2>&1; echo "ncu C=$C rc=$?"
done
