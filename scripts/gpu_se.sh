mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x -k "fp32 or f32 or se or SE or layout or backward" > gpurun_out/se_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/se_tests.log
timeout 600 python bench.py --workload se --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/se.json 2> gpurun_out/se.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/se.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value']/1e6, d['roofline_operator'])"
