mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_kernel -s 0 -c 2 -o gpurun_out/prof_fft python scripts/fftprof.py > gpurun_out/ncu_fft_full.log 2>&1; echo "ncu rc=$?"
