# round 2, batch bf: count-contract / per-chunk histogram with ONE 1024-thread worker per SM (sets of 32 KB, all
# below 96 KB) vs two 512-thread workers (product)
set -x
mkdir -p gpurun_out/bf
for v in prod w1024s3 w1024s2; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist --dump gpurun_out/bf/${v}_150.npz $lib > gpurun_out/bf/${v}_150.log 2>&1; echo "$v 150"; cat gpurun_out/bf/${v}_150.log
  timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only fused,score4,hist_chunks $lib > gpurun_out/bf/${v}_1500.log 2>&1; echo "$v 1500"; cat gpurun_out/bf/${v}_1500.log
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks --dump gpurun_out/bf/${v}_1m.npz $lib > gpurun_out/bf/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/bf/${v}_1m.log
done
python - <<'PY'
import numpy as np
for suf in ("150", "1m"):
    a = np.load(f"gpurun_out/bf/prod_{suf}.npz")
    for v in ("w1024s3", "w1024s2"):
        b = np.load(f"gpurun_out/bf/{v}_{suf}.npz")
        print(v, suf, all(np.array_equal(a[k], b[k]) for k in a.files))
PY
rm -f gpurun_out/bf/*.npz
