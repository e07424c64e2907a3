set -x
mkdir -p gpurun_out/z
MOEPLACE_PEER_NO_MULTICAST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/time_allreduce.py > gpurun_out/z/ar_p2p.log 2>&1; echo "ar rc=$?"; tail -1 gpurun_out/z/ar_p2p.log
MOEPLACE_PEER_NO_MULTICAST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 tools/check_multigpu.py > gpurun_out/z/check_p2p.log 2>&1; echo "check rc=$?"; tail -1 gpurun_out/z/check_p2p.log
