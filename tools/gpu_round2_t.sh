# round 2, batch t: warp-private histogram bins (microbench10)
set -x
mkdir -p gpurun_out/t
for a in "1.2 0" "1.2 1" "0 0" "2.0 0"; do ./tools/microbench10 $a >> gpurun_out/t/mb10.txt 2>&1; done
