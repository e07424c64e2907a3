# round 2, batch at: kernel table on the two-set build (C = 150, 1500) + weak scaling 1/2/4 GPUs (peer all-reduce)
set -x
mkdir -p gpurun_out/at
timeout 900 python tools/time_kernels.py --reps 10 --out gpurun_out/at/kernels_150.json > gpurun_out/at/kernels_150.log 2>&1; echo "tk rc=$?"
timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only hist,score1,score2,score4,fused,fused2,fused4,hist_chunks > gpurun_out/at/kernels_1500.log 2>&1; echo "tk1500 rc=$?"
timeout 600 python tools/time_kernels.py --reps 10 --only fused2,fused4,score1_count,score2_count > gpurun_out/at/kernels_150b.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/at/bench1.json 2> gpurun_out/at/bench1.err; echo "b1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $N > gpurun_out/at/bench$N.json 2> gpurun_out/at/bench$N.err; echo "b$N rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus $N --collective nccl > gpurun_out/at/bench${N}_nccl.json 2> gpurun_out/at/bench${N}_nccl.err; echo "b${N}nccl rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 tools/time_allreduce.py > gpurun_out/at/ar_4.log 2>&1; echo "ar rc=$?"
