# round 2, batch cf: single staggered worker vs two 512-thread workers under concurrent multi-GPU load (1 and 2 GPUs)
set -x
mkdir -p gpurun_out/cf
for v in prod nosingle; do
  [ $v != prod ] && export MOEPLACE_EXPERIMENT_LIB=$PWD/paper_2508_09229_b200/lib/libexp_$v.so
  timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/cf/${v}_n1.json 2> gpurun_out/cf/${v}_n1.err; echo "$v n1 rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --no-e2e > gpurun_out/cf/${v}_n2.json 2> gpurun_out/cf/${v}_n2.err; echo "$v n2 rc=$?"
  timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/cf/${v}_n1b.json 2> gpurun_out/cf/${v}_n1b.err; echo "$v n1b rc=$?"
  unset MOEPLACE_EXPERIMENT_LIB
done
