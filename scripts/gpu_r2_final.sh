# round-2 evidence pass: every bench workload at N=1, the kernel micro-benchmarks, the default
# bench's ncu launch list and one ncu --set full capture of its mixer
mkdir -p gpurun_out
for w in mr se li li_f32 stripe mr_train; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 > gpurun_out/final_$w.json 2> gpurun_out/final_$w.err
  echo "$w rc=$?"; cut -c1-300 gpurun_out/final_$w.json
done
timeout 900 python scripts/bench_kernels.py > gpurun_out/final_kernels.jsonl 2> gpurun_out/final_kernels.err; echo "kernels rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:two_stage_kernel -c 1 -o gpurun_out/final_mr_mixer \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu mr rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:two_stage_kernel -c 1 -o gpurun_out/final_li_mixer \
  python bench.py --workload li --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu li rc=$?"
