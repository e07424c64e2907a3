set -x
mkdir -p gpurun_out/af
for N in 10000000 9830400 9838592; do
  timeout 600 python tools/time_kernels.py --tokens $N --chunks 150 --reps 10 --only fused,hist_chunks,score4 > gpurun_out/af/n$N.log 2>&1
done
timeout 600 python tools/time_kernels.py --tokens 9830400 --chunks 1 --reps 10 --only fused,hist_chunks > gpurun_out/af/n9830400_c1.log 2>&1
