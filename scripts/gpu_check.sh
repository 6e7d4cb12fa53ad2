mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload stripe > gpurun_out/bench_stripe.json 2> gpurun_out/bench_stripe.err; echo "bench stripe rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_stripe.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value']/1e6, d['phases_ms'], d['roofline_operator']['frac'])"
