set -x
mkdir -p gpurun_out/ao
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum
for v in one512 two512; do
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/ao/t_$v.log 2>&1
  MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_$v.so timeout 600 ncu --metrics $M -k regex:pipe_kernel -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 --chunks 150 > gpurun_out/ao/ncu_$v.csv 2>&1
done
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist > gpurun_out/ao/t_base.log 2>&1
