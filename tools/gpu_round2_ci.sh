# round 2, batch ci: final 1/2/4-GPU weak (config 2) and strong (config 5) scaling, peer and NCCL all-reduce, reference arm
set -x
mkdir -p gpurun_out/ci
timeout 900 python bench.py --no-cpu > gpurun_out/ci/w2_n1.json 2> gpurun_out/ci/w2_n1.err; echo "w2n1 rc=$?"
timeout 900 python bench.py --workload 5 --no-cpu > gpurun_out/ci/w5_n1.json 2> gpurun_out/ci/w5_n1.err; echo "w5n1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $N > gpurun_out/ci/w2_n$N.json 2> gpurun_out/ci/w2_n$N.err; echo "w2n$N rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus $N --collective nccl > gpurun_out/ci/w2_n${N}_nccl.json 2> gpurun_out/ci/w2_n${N}_nccl.err; echo "w2n${N}nccl rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29593 bench.py --workload 5 --gpus $N > gpurun_out/ci/w5_n$N.json 2> gpurun_out/ci/w5_n$N.err; echo "w5n$N rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29594 bench.py --impl reference --gpus 4 > gpurun_out/ci/ref_n4.json 2> gpurun_out/ci/ref_n4.err; echo "ref4 rc=$?"
