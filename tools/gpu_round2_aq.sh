# round 2, batch aq: 2 vs 3 replica sets by piece length; full parity run on the product build
set -x
mkdir -p gpurun_out/aq
timeout 1500 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -x -q -p no:cacheprovider > gpurun_out/aq/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/aq/tests.log
for C in 150 300 450 600 900 1500; do
  for v in f2 f3; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/aq/t_${v}_$C.log 2>&1
  done
done
for v in f2 f3; do timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/aq/t_${v}_1m.log 2>&1; done
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist > gpurun_out/aq/t_prod_150.log 2>&1
