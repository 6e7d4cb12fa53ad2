mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x > gpurun_out/mr_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/mr_tests.log
timeout 300 python scripts/trace_ts.py mixer > gpurun_out/trace_mr_mixer.txt 2>&1; echo "trace rc=$?"; grep -E "period|tiles" gpurun_out/trace_mr_mixer.txt | head -3
timeout 300 python scripts/bench_kernels.py --which mr > gpurun_out/bk_mr.txt 2>&1; cat gpurun_out/bk_mr.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mr.json 2> gpurun_out/mr.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/mr.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_ms'])"
