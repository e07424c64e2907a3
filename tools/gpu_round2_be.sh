# round 2, batch be: token_hops TMA-ring shapes (threads, tokens per thread, ring slots) vs the round-1 kernel
set -x
mkdir -p gpurun_out/be
for v in tok0 tokt_512_8_4 tokt_512_8_3 tokt_1024_4_2 tokt_512_4_4; do
  timeout 600 python tools/time_kernels.py --reps 10 --only token_hops --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/be/$v.log 2>&1; echo "$v"; cat gpurun_out/be/$v.log
done
timeout 600 python tools/time_kernels.py --reps 10 --only token_hops > gpurun_out/be/prod.log 2>&1; echo prod; cat gpurun_out/be/prod.log
