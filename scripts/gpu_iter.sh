# quick iteration: parity tests for the kernels + micro-bench (both converter-warp configs)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -5
for cw in 8 12; do HY_TS_CONV_WARPS=$cw timeout 300 python scripts/bench_kernels.py --which ${WHICH:-all} | sed "s/^/cw=$cw /"; done
