mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 300 -p no:cacheprovider -k "fft" > gpurun_out/fft_tests.log 2>&1; echo "fft tests rc=$?"; tail -15 gpurun_out/fft_tests.log
timeout 600 python scripts/bench_kernels.py --which fft > gpurun_out/bk_fft.txt 2>&1; echo "bk fft rc=$?"; cat gpurun_out/bk_fft.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fft.csv python scripts/fftprof.py > gpurun_out/ncu_fft.log 2>&1; echo "ncu rc=$?"
