# round 2, batch ca: product with the single staggered worker for long pieces + piece-end bytes after the vectors
set -x
mkdir -p gpurun_out/ca
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ca/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ca/pytest.log
for C in 1 50 150 300 600 1500; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,score8,hist_chunks > gpurun_out/ca/k_$C.log 2>&1; echo "C=$C"; cat gpurun_out/ca/k_$C.log
done
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks > gpurun_out/ca/k_1m.log 2>&1; echo "1m"; cat gpurun_out/ca/k_1m.log
timeout 600 python tools/time_kernels.py --reps 10 --only hist > gpurun_out/ca/k_hist.log 2>&1; cat gpurun_out/ca/k_hist.log
timeout 900 python bench.py > gpurun_out/ca/bench.json 2> gpurun_out/ca/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --workload 3 --no-cpu > gpurun_out/ca/bench_wl3.json 2> gpurun_out/ca/bench_wl3.err; echo "wl3 rc=$?"
timeout 900 python bench.py --workload 4 --no-cpu > gpurun_out/ca/bench_wl4.json 2> gpurun_out/ca/bench_wl4.err; echo "wl4 rc=$?"
