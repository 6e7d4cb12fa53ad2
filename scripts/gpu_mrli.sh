mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t.log
timeout 300 python scripts/bench_kernels.py --which mr > gpurun_out/bk_mr.txt 2>&1; cat gpurun_out/bk_mr.txt
timeout 300 python scripts/bench_kernels.py --which li > gpurun_out/bk_li.txt 2>&1; cat gpurun_out/bk_li.txt
timeout 300 python scripts/trace_ts.py mixer 2>&1 | grep period
timeout 300 python scripts/trace_li.py mixer 2>&1 | grep -E "period E_done|period M_E"
