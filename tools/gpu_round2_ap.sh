set -x
mkdir -p gpurun_out/ap
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_sets2.so timeout 900 python -m pytest tests/test_gpu_algos.py tests/test_gpu_properties.py -x -q -p no:cacheprovider -k "algorithms or stress" > gpurun_out/ap/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ap/tests.log
for C in 150 1500; do
for v in sets2 one512; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks,hist --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/ap/t_${v}_$C.log 2>&1
done
timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,hist_chunks,hist > gpurun_out/ap/t_base_$C.log 2>&1
done
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks --lib paper_2508_09229_b200/lib/libexp_sets2.so > gpurun_out/ap/t_sets2_1m.log 2>&1
timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks > gpurun_out/ap/t_base_1m.log 2>&1
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_sets2.so timeout 600 ncu --metrics $M -k regex:pipe_kernel -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 --chunks 150 > gpurun_out/ap/ncu_sets2.csv 2>&1
