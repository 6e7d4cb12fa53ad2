mkdir -p gpurun_out
timeout 900 python scripts/bench_kernels.py > gpurun_out/kernels_all.jsonl 2> gpurun_out/kernels_all.err; echo "bk rc=$?"; cat gpurun_out/kernels_all.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:causal_conv -s 2 -c 1 -o gpurun_out/prof_feat python scripts/featprof.py > gpurun_out/ncu_feat.log 2>&1; echo "ncu feat rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_kernel -s 1 -c 1 -o gpurun_out/prof_fftrow python scripts/fftprof.py > gpurun_out/ncu_fftrow.log 2>&1; echo "ncu fft rc=$?"
