# round 2, batch bd: token_hops with the TMA ring (K = 8) - parity + timing vs the round-1 kernel
set -x
mkdir -p gpurun_out/bd
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "token_hops" > gpurun_out/bd/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bd/tests.log
timeout 600 python tools/time_kernels.py --reps 10 --only token_hops > gpurun_out/bd/tma.log 2>&1; cat gpurun_out/bd/tma.log
timeout 600 python tools/time_kernels.py --reps 10 --only token_hops --lib paper_2508_09229_b200/lib/libexp_tok0.so > gpurun_out/bd/old.log 2>&1; cat gpurun_out/bd/old.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"token_hops_tma" -c 1 -o gpurun_out/bd/tok python tools/time_kernels.py --reps 1 --only token_hops > gpurun_out/bd/ncu.log 2>&1; echo "ncu rc=$?"
