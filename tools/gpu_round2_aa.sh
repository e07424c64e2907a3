set -x
mkdir -p gpurun_out/aa
MP_STRESS_EXAMPLES=25 timeout 1500 python -m pytest tests/test_gpu_properties.py -x -q -p no:cacheprovider -k "views_stress or multi_cta_stress or dedup_warp" > gpurun_out/aa/stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/aa/stress.log
