set -x
mkdir -p gpurun_out/as
timeout 900 python bench.py --workload 4 > gpurun_out/as/bench_wl4.json 2> gpurun_out/as/bench_wl4.err; echo "bench4 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/as/ref.json 2> gpurun_out/as/ref.err; echo "ref rc=$?"
