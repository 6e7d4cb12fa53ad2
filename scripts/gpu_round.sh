# Round evidence: all GPU tests, bench lines for every single-GPU workload, LI launch list + ncu
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for W in mr se li stripe mr_train; do
  timeout 900 python bench.py --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "bench $W rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_$W.json').read().strip().splitlines()[-1]); print('$W', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'Mtok/s', 'roof', round(d['roofline']['frac'],3), d['roofline']['launch_ms'], 'e2e', round(d['e2e']['value']/1e6,3), 'cpu', d.get('cpu_baseline',{}).get('value'))"
done
CMD="python bench.py --workload li --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_li.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_li.csv $CMD > gpurun_out/ncu_launch_li.log 2>&1; echo "ncu launches li rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:two_stage_kernel -s 3 -c 1 -o gpurun_out/prof_li $CMD > gpurun_out/ncu_full_li.log 2>&1; echo "ncu full li rc=$?"
