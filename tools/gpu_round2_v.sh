# round 2, batch v: peer-memory (NVLS multimem) sum of the packed result vs NCCL all_reduce, 2 and 4 GPUs
set -x
mkdir -p gpurun_out/v
N=${N:-4}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 tools/check_multigpu.py > gpurun_out/v/check_$N.log 2>&1; echo "check rc=$?"; tail -2 gpurun_out/v/check_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus $N --no-e2e --no-cpu > gpurun_out/v/peer_$N.json 2> gpurun_out/v/peer_$N.err; echo "peer rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus $N --no-e2e --no-cpu --collective nccl > gpurun_out/v/nccl_$N.json 2> gpurun_out/v/nccl_$N.err; echo "nccl rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 tools/time_allreduce.py > gpurun_out/v/ar_$N.log 2>&1; echo "ar rc=$?"; cat gpurun_out/v/ar_$N.log | tail -4
