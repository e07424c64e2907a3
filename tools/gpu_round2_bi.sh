# round 2, batch bi: cross-piece prefetch of the next piece's first 4 vectors per thread (MP_PIPE_XPF=1) vs product
set -x
mkdir -p gpurun_out/bi
for v in prod xpf; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist --dump gpurun_out/bi/${v}_150.npz $lib > gpurun_out/bi/${v}_150.log 2>&1; echo "$v 150"; cat gpurun_out/bi/${v}_150.log
  timeout 600 python tools/time_kernels.py --chunks 1500 --reps 10 --only fused,score4,hist_chunks $lib > gpurun_out/bi/${v}_1500.log 2>&1; echo "$v 1500"; cat gpurun_out/bi/${v}_1500.log
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks --dump gpurun_out/bi/${v}_1m.npz $lib > gpurun_out/bi/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/bi/${v}_1m.log
done
python - <<'PY'
import numpy as np
for suf in ("150", "1m"):
    a, b = np.load(f"gpurun_out/bi/prod_{suf}.npz"), np.load(f"gpurun_out/bi/xpf_{suf}.npz")
    print(suf, all(np.array_equal(a[k], b[k]) for k in a.files))
PY
rm -f gpurun_out/bi/*.npz
