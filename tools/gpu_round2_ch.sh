# round 2, batch ch: kernel shape from the non-empty chunks (shards keep the global chunk list, clipped)
set -x
mkdir -p gpurun_out/ch
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ch/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ch/pytest.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/ch/w2_n1.json 2> gpurun_out/ch/w2_n1.err; echo "w2n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --no-e2e > gpurun_out/ch/w2_n2.json 2> gpurun_out/ch/w2_n2.err; echo "w2n2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 bench.py --workload 5 --gpus 2 --no-e2e > gpurun_out/ch/w5_n2.json 2> gpurun_out/ch/w5_n2.err; echo "w5n2 rc=$?"
