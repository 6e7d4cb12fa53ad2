# Final evidence: smoke, all GPU tests, bench lines for every single-GPU workload, the default
# command's launch list and ncu capture of the MR mixer
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for W in mr se li stripe mr_train; do
  timeout 900 python bench.py --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "bench $W rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_$W.json').read().strip().splitlines()[-1]); print('$W', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'Mtok/s', 'roof', round(d['roofline']['frac'],3), round(d['roofline']['launch_ms'],4), 'e2e', round(d['e2e']['value']/1e6,3), 'clk', d['clocks'])"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:two_stage_kernel -s 2 -c 1 -o gpurun_out/prof_mr $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
