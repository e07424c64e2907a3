set -x
mkdir -p gpurun_out/am
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,gpu__time_duration.sum
for st in 0 1 2; do
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_set$st.so timeout 600 ncu --metrics $M -k regex:"pipe_kernel" -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 --chunks 150 > gpurun_out/am/ncu_set$st.csv 2>&1
done
