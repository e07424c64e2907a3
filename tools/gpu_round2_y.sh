# round 2, batch y: ncu of the per-chunk histogram at config-4 size (1M tokens, 150 chunks)
set -x
mkdir -p gpurun_out/y
timeout 300 python tools/prof_kernels.py --tokens 1000000 --chunks 150 --which hist_chunks --reps 1 > gpurun_out/y/plain.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -c 1 -o gpurun_out/y/hc python tools/prof_kernels.py --tokens 1000000 --chunks 150 --which hist_chunks --reps 1 > gpurun_out/y/ncu.log 2>&1; echo "ncu rc=$?"
