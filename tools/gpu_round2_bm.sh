# round 2, batch bm: count-contract sets in [0, 128 KB) with a larger shared-memory allocation / carveout (is set 1 then fast?)
set -x
mkdir -p gpurun_out/bm
for v in prod alloc192 alloc224 carve100; do
  lib=""; [ $v != prod ] && lib="--lib paper_2508_09229_b200/lib/libexp_$v.so"
  timeout 600 python tools/time_kernels.py --chunks 150 --reps 10 --only fused,score4,hist_chunks,hist $lib > gpurun_out/bm/$v.log 2>&1; echo "$v"; cat gpurun_out/bm/$v.log
done
