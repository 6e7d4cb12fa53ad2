# SE mixer iteration: parity tests, kernel microbench, one ncu capture of the fp32 SE kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "se_mixer" --timeout 300 -p no:cacheprovider > gpurun_out/pytest_se.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_se.log
timeout 300 python scripts/bench_kernels.py --which se > gpurun_out/bk_se.txt 2>&1; echo "bk se rc=$?"; cat gpurun_out/bk_se.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:se_stream_kernel -s 5 -c 1 -o gpurun_out/prof_se python scripts/bench_kernels.py --which se > gpurun_out/ncu_se.log 2>&1; echo "ncu se rc=$?"; tail -3 gpurun_out/ncu_se.log
