# round 2, batch ck: the gather (stream_kernel) with its piece-end bytes counted after the vectors
set -x
mkdir -p gpurun_out/ck
for v in prod nofix; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 150 1500; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score1,score1_gather,fused_gather,score2_gather --dump gpurun_out/ck/${v}_$C.npz $lib > gpurun_out/ck/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/ck/${v}_$C.log
  done
done
python - <<'PY'
import numpy as np
for C in (150, 1500):
    a, b = np.load(f"gpurun_out/ck/prod_{C}.npz"), np.load(f"gpurun_out/ck/nofix_{C}.npz")
    print(C, all(np.array_equal(a[k], b[k]) for k in a.files))
PY
rm -f gpurun_out/ck/*.npz
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/ck/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ck/tests.log
