set -x
mkdir -p gpurun_out/ai
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,gpu__time_duration.sum
run() { name=$1; shift; timeout 900 ncu --metrics $M -k regex:pipe_kernel -c 1 --csv python tools/prof_kernels.py --which fused --reps 1 "$@" > gpurun_out/ai/$name.csv 2>&1; }
run c150 --chunks 150
run c150_aligned --chunks 150 --tokens 9830400
run c1 --chunks 1
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_cap.so run c1_cap533k --chunks 1
MOEPLACE_EXPERIMENT_LIB=paper_2508_09229_b200/lib/libexp_cap2.so run c1_cap512k --chunks 1
for f in c1 c150; do :; done
timeout 600 python tools/time_kernels.py --chunks 1 --reps 10 --only fused --lib paper_2508_09229_b200/lib/libexp_cap.so > gpurun_out/ai/t_c1_cap533k.log 2>&1
timeout 600 python tools/time_kernels.py --chunks 1 --reps 10 --only fused --lib paper_2508_09229_b200/lib/libexp_cap2.so > gpurun_out/ai/t_c1_cap512k.log 2>&1
