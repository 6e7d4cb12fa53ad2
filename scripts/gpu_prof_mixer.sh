timeout 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -20
CMD="python scripts/bench_kernels.py --which mr"
$CMD > gpurun_out/plain_mixer.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:two_stage_kernel -s 3 -c 1 -o gpurun_out/prof_mixer $CMD > gpurun_out/ncu_mixer.log 2>&1; echo "ncu rc=$?"
