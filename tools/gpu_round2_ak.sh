# round 2, batch ak: staggered replica sets in pipe_kernel (ATOMS aliasing between sets)
set -x
mkdir -p gpurun_out/ak
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,gpu__time_duration.sum
for v in skew256 skew512 skew1280 skew4096; do
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/ak/t_$v.log 2>&1
  MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_$v.so timeout 600 ncu --metrics $M -k regex:pipe_kernel -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 --chunks 150 > gpurun_out/ak/ncu_$v.csv 2>&1
done
timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks > gpurun_out/ak/t_base.log 2>&1
