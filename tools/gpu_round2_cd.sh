# round 2, batch cd: a piece's remainder vectors alternate between the worker halves (thread index rotated by half a
# worker every other piece)
set -x
mkdir -p gpurun_out/cd
for v in prod rot; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  for C in 50 150 300 1500; do
    timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only fused,score4,score8 --dump gpurun_out/cd/${v}_$C.npz $lib > gpurun_out/cd/${v}_$C.log 2>&1; echo "$v C=$C"; cat gpurun_out/cd/${v}_$C.log
  done
  timeout 600 python tools/time_kernels.py --tokens 1000000 --chunks 150 --reps 20 --only hist_chunks $lib > gpurun_out/cd/${v}_1m.log 2>&1; echo "$v 1m"; cat gpurun_out/cd/${v}_1m.log
done
python - <<'PY'
import numpy as np
for C in (50, 150, 300, 1500):
    a, b = np.load(f"gpurun_out/cd/prod_{C}.npz"), np.load(f"gpurun_out/cd/rot_{C}.npz")
    print(C, all(np.array_equal(a[k], b[k]) for k in a.files))
PY
rm -f gpurun_out/cd/*.npz
