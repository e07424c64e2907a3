set -x
mkdir -p gpurun_out/al
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,gpu__time_duration.sum
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,hist_chunks --lib paper_2508_09229_b200/lib/libexp_flush0.so > gpurun_out/al/t_flush0.log 2>&1
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_flush0.so timeout 600 ncu --metrics $M -k regex:"stream_kernel|pipe_kernel" -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 --chunks 150 > gpurun_out/al/ncu_flush0.csv 2>&1
