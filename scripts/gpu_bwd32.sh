mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_backward_kernels.py -q --timeout 300 -p no:cacheprovider > gpurun_out/bwd_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/bwd_tests.log
timeout 600 python scripts/bench_backward.py > gpurun_out/bk_bwd.txt 2>&1; echo "bk rc=$?"; cut -c1-200 gpurun_out/bk_bwd.txt
