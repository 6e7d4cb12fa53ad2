mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cp.py -q --timeout 600 -p no:cacheprovider > gpurun_out/cp_tests.log 2>&1; echo "cp tests rc=$?"; tail -3 gpurun_out/cp_tests.log
W=mr STEPS=20 bash scripts/gpu_cp_scale.sh
