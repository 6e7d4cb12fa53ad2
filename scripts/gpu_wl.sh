# one workload: bench line + launch list (usage: WL=se bash scripts/gpu_wl.sh)
mkdir -p gpurun_out
WL=${WL:-se}
python bench.py --workload $WL > gpurun_out/bench_$WL.json 2> gpurun_out/bench_$WL.err; echo "bench $WL rc=$?"; cat gpurun_out/bench_$WL.json; tail -3 gpurun_out/bench_$WL.err
CMD="python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_$WL.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$WL.csv $CMD > gpurun_out/ncu_launch_$WL.log 2>&1; echo "ncu launches rc=$?"
