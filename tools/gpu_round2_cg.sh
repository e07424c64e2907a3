# round 2, batch cg: kernel shape from the chunks' true length (shards of a larger trace), GPU suite, 1/2/4-GPU weak + strong scaling
set -x
mkdir -p gpurun_out/cg
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/cg/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/cg/pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/cg/w2_n1.json 2> gpurun_out/cg/w2_n1.err; echo "w2n1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N > gpurun_out/cg/w2_n$N.json 2> gpurun_out/cg/w2_n$N.err; echo "w2n$N rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29572 bench.py --workload 5 --gpus $N > gpurun_out/cg/w5_n$N.json 2> gpurun_out/cg/w5_n$N.err; echo "w5n$N rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29573 bench.py --gpus 4 --collective nccl > gpurun_out/cg/w2_n4_nccl.json 2> gpurun_out/cg/w2_n4_nccl.err; echo "w2n4nccl rc=$?"
timeout 900 python bench.py --workload 5 --no-cpu > gpurun_out/cg/w5_n1.json 2> gpurun_out/cg/w5_n1.err; echo "w5n1 rc=$?"
