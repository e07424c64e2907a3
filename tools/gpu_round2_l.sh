# round 2, batch l: ATOMS wavefronts vs row pitch (microbench9) + ncu conflict counters
set -x
mkdir -p gpurun_out/l
for s in 1.2 0 2.0; do ./tools/microbench9 $s >> gpurun_out/l/mb9.txt 2>&1; done
timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum -k regex:hist_kernel -s 15 -c 5 --csv ./tools/microbench9 1.2 > gpurun_out/l/mb9_ncu.csv 2>&1; echo "ncu rc=$?"
