# round 2, batch q: 2/4-GPU weak scaling (config 2) and config-5 strong scaling with the round-2 kernels
set -x
mkdir -p gpurun_out/q
run() { n=$1; shift; timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
run 2 > gpurun_out/q/w2_n2.json 2> gpurun_out/q/w2_n2.err; echo "w2 n2 rc=$?"
run 4 > gpurun_out/q/w2_n4.json 2> gpurun_out/q/w2_n4.err; echo "w2 n4 rc=$?"
timeout 1200 python bench.py --workload 5 --no-e2e > gpurun_out/q/w5_n1.json 2> gpurun_out/q/w5_n1.err; echo "w5 n1 rc=$?"
run 4 --workload 5 > gpurun_out/q/w5_n4.json 2> gpurun_out/q/w5_n4.err; echo "w5 n4 rc=$?"
run 4 --impl reference > gpurun_out/q/ref_n4.json 2> gpurun_out/q/ref_n4.err; echo "ref n4 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/check_multigpu.py > gpurun_out/q/check.log 2>&1; echo "check rc=$?"
