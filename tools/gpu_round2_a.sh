set -x
mkdir -p gpurun_out/bench_data
for w in 2 3 4; do
  timeout 900 python bench.py --workload $w --write-fixtures bench_data --no-e2e --no-cpu --steps 3 --warmup 3 --sustained-s 0 > gpurun_out/fx_$w.json 2> gpurun_out/fx_$w.err; echo "fx $w rc=$?"
done
cp bench_data/*.npz gpurun_out/bench_data/
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
