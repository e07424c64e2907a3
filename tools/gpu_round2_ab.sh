set -x
mkdir -p gpurun_out/ab
for C in 1 10 50 150 300; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks,hist > gpurun_out/ab/c$C.log 2>&1; echo "C=$C rc=$?"
done
