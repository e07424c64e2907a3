# round 2, batch bb: nibble tables in the segmented gather (W = 2 / 4, max_p <= 15): parity + timing vs u8 tables
set -x
mkdir -p gpurun_out/bb
timeout 1200 python -m pytest tests/test_gpu_algos.py tests/test_gpu_parity.py tests/test_gpu_properties.py -x -q -p no:cacheprovider > gpurun_out/bb/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bb/tests.log
for C in 71429 15000 3000; do
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score2_seg,fused2_seg,score4_seg,fused4_seg --dump gpurun_out/bb/n_$C.npz > gpurun_out/bb/n_$C.log 2>&1; echo "nib $C"; cat gpurun_out/bb/n_$C.log
  timeout 600 python tools/time_kernels.py --chunks $C --reps 10 --only score2_seg,fused2_seg,score4_seg,fused4_seg --dump gpurun_out/bb/u_$C.npz --lib paper_2508_09229_b200/lib/libexp_nonib.so > gpurun_out/bb/u_$C.log 2>&1; echo "u8 $C"; cat gpurun_out/bb/u_$C.log
done
timeout 600 python tools/time_kernels.py --chunks 3000 --reps 5 --only score4_count,fused4_count,score2_count,fused2_count > gpurun_out/bb/count_3000.log 2>&1; cat gpurun_out/bb/count_3000.log
python - <<'PY'
import numpy as np
for C in (71429, 15000, 3000):
    a, b = np.load(f"gpurun_out/bb/n_{C}.npz"), np.load(f"gpurun_out/bb/u_{C}.npz")
    print(C, {k: bool(np.array_equal(a[k], b[k])) for k in a.files})
PY
rm -f gpurun_out/bb/*.npz
