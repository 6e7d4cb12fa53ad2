mkdir -p gpurun_out
for W in mr li se; do
  timeout 900 python bench.py --workload $W --group-size 16 --no-cpu-baseline > gpurun_out/bench_${W}_g16.json 2> gpurun_out/bench_${W}_g16.err; echo "$W g16 rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_${W}_g16.json').read().strip().splitlines()[-1]); print('$W g16', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'Mtok/s roof', round(d['roofline']['frac'],3), round(d['roofline']['launch_ms'],4))"
done
