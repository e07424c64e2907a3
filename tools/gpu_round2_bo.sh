# round 2, batch bo: count-contract with 2 x 256-thread workers per SM (up to 128 registers per thread) vs 2 x 512
set -x
mkdir -p gpurun_out/bo
for v in prod wt256u32 wt256u16; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks --dump gpurun_out/bo/${v}.npz $lib > gpurun_out/bo/$v.log 2>&1; echo "$v"; cat gpurun_out/bo/$v.log
  timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only fused,score4,hist_chunks $lib > gpurun_out/bo/${v}_1500.log 2>&1; cat gpurun_out/bo/${v}_1500.log
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks $lib > gpurun_out/bo/${v}_1m.log 2>&1; cat gpurun_out/bo/${v}_1m.log
done
python - <<'PY'
import numpy as np
a = np.load("gpurun_out/bo/prod.npz")
for v in ("wt256u32", "wt256u16"):
    b = np.load(f"gpurun_out/bo/{v}.npz"); print(v, all(np.array_equal(a[k], b[k]) for k in a.files))
PY
rm -f gpurun_out/bo/*.npz
