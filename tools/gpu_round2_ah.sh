set -x
mkdir -p gpurun_out/ah
for v in noflush oneset; do
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/ah/t_$v.log 2>&1
  MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_$v.so timeout 900 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,gpu__time_duration.sum -k regex:pipe_kernel -c 1 --csv python tools/prof_kernels.py --chunks 150 --which fused --reps 1 > gpurun_out/ah/ncu_$v.csv 2>&1
done
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused > gpurun_out/ah/t_base.log 2>&1
