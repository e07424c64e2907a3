set -x
mkdir -p gpurun_out/aj
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,gpu__time_duration.sum
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_oneset.so timeout 600 ncu --metrics $M -k regex:pipe_kernel -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 --chunks 1 > gpurun_out/aj/oneset.csv 2>&1; echo "rc=$?"
