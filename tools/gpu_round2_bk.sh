# round 2, batch bk: launch lists (config 2 / 3 / 4 bench steps) and ncu --set full of the histogram and W = 8 kernels
set -x
mkdir -p gpurun_out/bk
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bk/launches_wl2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > gpurun_out/bk/l2.log 2>&1; echo "l2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bk/launches_wl3.csv python bench.py --workload 3 --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > gpurun_out/bk/l3.log 2>&1; echo "l3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bk/launches_wl4.csv python bench.py --workload 4 --steps 2 --warmup 3 --no-e2e --no-cpu --sustained-s 0 > gpurun_out/bk/l4.log 2>&1; echo "l4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pipe_kernel" -c 3 -o gpurun_out/bk/pipe python tools/time_kernels.py --reps 1 --only hist,score8,fused > gpurun_out/bk/ncu.log 2>&1; echo "ncu rc=$?"
