# SE micro-bench incl. the routed bf16 (tcgen05) SE mixer, plus the GPU tests on the final library
mkdir -p gpurun_out
timeout 600 python scripts/bench_kernels.py --which se > gpurun_out/kernels_se4.jsonl 2>&1; echo "bk rc=$?"; cut -c1-200 gpurun_out/kernels_se4.jsonl
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu5.log
