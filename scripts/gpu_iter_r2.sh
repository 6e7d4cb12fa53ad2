# iteration pass: selected tests (PT_K), the row-shift descriptor probe, selected bench workloads,
# and one ncu --set full capture of NCU_KERNEL in workload NCU_WL
mkdir -p gpurun_out
if [ -n "$PT_K" ]; then
  timeout ${PT_TIMEOUT:-1200} python -m pytest tests -m gpu -q -rs ${PT_X:-} -k "$PT_K" > gpurun_out/pytest_iter.log 2>&1
  echo "pytest rc=$?"; tail -25 gpurun_out/pytest_iter.log
fi
[ -n "$PROBE" ] && timeout 120 python $PROBE 2>&1 | tail -5
[ -n "$KBENCH" ] && timeout 600 python scripts/bench_kernels.py --which $KBENCH 2>&1 | tail -20
for w in $WLS; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 ${BENCH_EXTRA:-} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"; cut -c1-1500 gpurun_out/bench_$w.json; tail -3 gpurun_out/bench_$w.err
done
if [ -n "$NCU_KERNEL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -c 1 -o gpurun_out/ncu_$NCU_TAG \
    python bench.py --workload $NCU_WL --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$NCU_TAG.log 2>&1
  echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$NCU_TAG.log
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$NCU_TAG.csv \
    python bench.py --workload $NCU_WL --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "launches rc=$?"
fi
