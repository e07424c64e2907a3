set -x
mkdir -p gpurun_out/an
./tools/microbench11 > gpurun_out/an/mb11.txt 2>&1; echo "rc=$?"
timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,gpu__time_duration.sum -k regex:hist_kernel -s 2 --csv ./tools/microbench11 > gpurun_out/an/ncu.csv 2>&1; echo "ncu rc=$?"
