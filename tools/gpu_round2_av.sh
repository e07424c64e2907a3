# round 2, batch av: segmented-gather flush variants at 140 tokens per chunk (packed u16 reduce-scatter,
# redux.sync, no global atomics) vs the product flush; hop sums compared across variants
set -x
mkdir -p gpurun_out/av
for v in seg_p0 seg_p1 seg_p2 seg_nored; do
  timeout 600 python tools/time_kernels.py --chunks 71429 --reps 10 --only score1_seg,fused_seg,score4_seg,fused4_seg --dump gpurun_out/av/$v.npz --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/av/t_$v.log 2>&1; echo "$v rc=$?"
  cat gpurun_out/av/t_$v.log
done
for v in seg_p0 seg_p1 seg_p2; do
  timeout 600 python tools/time_kernels.py --chunks 15000 --reps 10 --only score1_seg,fused_seg,score4_seg --dump gpurun_out/av/${v}_15k.npz --lib paper_2508_09229_b200/lib/libexp_$v.so > gpurun_out/av/t15k_$v.log 2>&1; cat gpurun_out/av/t15k_$v.log
done
python - <<'PY'
import numpy as np
for suf in ("", "_15k"):
    a = np.load(f"gpurun_out/av/seg_p0{suf}.npz")
    for v in ("seg_p1", "seg_p2"):
        b = np.load(f"gpurun_out/av/{v}{suf}.npz")
        print(v, suf, {k: bool(np.array_equal(a[k], b[k])) for k in a.files})
PY
rm -f gpurun_out/av/*.npz
