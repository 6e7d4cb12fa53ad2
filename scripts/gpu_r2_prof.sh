bash scripts/gpu_sanitize.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_conv_kernel -c 1 -o gpurun_out/ncu_li_conv python scripts/bench_kernels.py --which li > gpurun_out/ncu_li_conv.log 2>&1; echo "ncu li_conv rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_conv_kernel -c 1 -o gpurun_out/ncu_kblock python scripts/bench_kernels.py --which kblock > gpurun_out/ncu_kblock.log 2>&1; echo "ncu kblock rc=$?"
timeout 600 python -m pytest tests -m gpu -q -k "li_scan_mixer" 2>&1 | tail -2
