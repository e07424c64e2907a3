# round 2, batch k: dedup with IMAD subtractions; new AUTO crossovers; full GPU suite
set -x
mkdir -p gpurun_out/k
for C in 150 15000 150000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 5 --only dedup > gpurun_out/k/dedup_$C.log 2>&1; echo "dedup $C rc=$?"
done
timeout 600 python tools/time_kernels.py --chunks 71429 --reps 5 --only fused,score1,score2,score4,fused2,fused4 > gpurun_out/k/auto_71429.log 2>&1; echo "auto rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/k/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/k/pytest.log
