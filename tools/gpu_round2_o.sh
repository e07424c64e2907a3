# round 2, batch o: register-resident generator (guide-table rank search)
set -x
mkdir -p gpurun_out/o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "generat or shard" > gpurun_out/o/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/o/tests.log
timeout 600 python tools/time_gen.py > gpurun_out/o/new.log 2>&1; echo "new rc=$?"
timeout 600 python tools/time_gen.py --lib paper_2508_09229_b200/lib/libexp_old.so > gpurun_out/o/old.log 2>&1; echo "old rc=$?"
