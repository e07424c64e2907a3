set -x
mkdir -p gpurun_out/w
N=${N:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 tools/time_allreduce.py > gpurun_out/w/ar_$N.log 2>&1; echo "ar rc=$?"; tail -2 gpurun_out/w/ar_$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29552 tools/check_multigpu.py > gpurun_out/w/check_$N.log 2>&1; echo "check rc=$?"; tail -1 gpurun_out/w/check_$N.log
