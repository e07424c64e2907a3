# round 2, batch n: ATOMS wavefronts vs trace structure (i.i.d. bytes / distinct 8-pick records / sorted records)
set -x
mkdir -p gpurun_out/n
for m in 0 1 2; do ./tools/microbench9 1.2 $m >> gpurun_out/n/mb9.txt 2>&1; done
for m in 0 1 2; do
timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum -k regex:hist_kernel -c 30 --csv ./tools/microbench9 1.2 $m > gpurun_out/n/ncu_$m.csv 2>&1; echo "ncu $m rc=$?"
done
