# round 2, batch bx: fused count-contract on one 1024-thread worker (3 x 32 KB sets) with the upper half started
# later by __nanosleep, so the halves' piece boundaries (load drains) are out of phase
set -x
mkdir -p gpurun_out/bx
for v in prod single single_st3 single_st6 single_st12; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,score8 --dump gpurun_out/bx/$v.npz $lib > gpurun_out/bx/$v.log 2>&1; echo "$v"; cat gpurun_out/bx/$v.log
done
python - <<'PY'
import numpy as np
a = np.load("gpurun_out/bx/prod.npz")
for v in ("single", "single_st3", "single_st6", "single_st12"):
    b = np.load(f"gpurun_out/bx/{v}.npz"); print(v, all(np.array_equal(a[k], b[k]) for k in a.files))
PY
rm -f gpurun_out/bx/*.npz
