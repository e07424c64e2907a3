# round 2, batch bc: config 5 (100M tokens, strong scaling) on 1 / 2 / 4 GPUs with the two-set kernel
set -x
mkdir -p gpurun_out/bc
timeout 900 python bench.py --workload 5 --no-cpu > gpurun_out/bc/w5_n1.json 2> gpurun_out/bc/w5_n1.err; echo "w5n1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 bench.py --workload 5 --gpus $N > gpurun_out/bc/w5_n$N.json 2> gpurun_out/bc/w5_n$N.err; echo "w5n$N rc=$?"
done
