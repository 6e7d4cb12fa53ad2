# Round-1 tail evidence: standalone kernel timings, SE e2e re-check, LI launch list + ncu of the LI mixer
mkdir -p gpurun_out
timeout 900 python scripts/bench_kernels.py > gpurun_out/kernels_all.jsonl 2> gpurun_out/kernels_all.err; echo "bk rc=$?"; cat gpurun_out/kernels_all.jsonl | cut -c1-220
for i in 1 2; do timeout 600 python bench.py --workload se --no-cpu-baseline > gpurun_out/bench_se_$i.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/bench_se_$i.json').read().strip().splitlines()[-1]); print('se', d['ms_per_step'], d['e2e'])"; done
CMD="python bench.py --workload li --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_li.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_li.csv $CMD > gpurun_out/ncu_launch_li.log 2>&1; echo "ncu launches li rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:two_stage_kernel -s 3 -c 1 -o gpurun_out/prof_li $CMD > gpurun_out/ncu_full_li.log 2>&1; echo "ncu full li rc=$?"
