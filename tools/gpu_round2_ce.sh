# round 2, batch ce: 1/2/4-GPU weak (config 2) and strong (config 5) scaling on the final kernel
set -x
mkdir -p gpurun_out/ce
timeout 900 python bench.py --no-cpu > gpurun_out/ce/w2_n1.json 2> gpurun_out/ce/w2_n1.err; echo "w2n1 rc=$?"
timeout 900 python bench.py --workload 5 --no-cpu > gpurun_out/ce/w5_n1.json 2> gpurun_out/ce/w5_n1.err; echo "w5n1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N > gpurun_out/ce/w2_n$N.json 2> gpurun_out/ce/w2_n$N.err; echo "w2n$N rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus $N --collective nccl > gpurun_out/ce/w2_n${N}_nccl.json 2> gpurun_out/ce/w2_n${N}_nccl.err; echo "w2n${N}nccl rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 bench.py --workload 5 --gpus $N > gpurun_out/ce/w5_n$N.json 2> gpurun_out/ce/w5_n$N.err; echo "w5n$N rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --impl reference --gpus 4 > gpurun_out/ce/ref_n4.json 2> gpurun_out/ce/ref_n4.err; echo "ref4 rc=$?"
