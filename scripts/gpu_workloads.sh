# every bench workload at N=1 (short runs), each under its own timeout
mkdir -p gpurun_out
for w in ${WORKLOADS:-mr se li stripe li_cp}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 ${EXTRA:---no-cpu-baseline} \
    > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"; cut -c1-400 gpurun_out/bench_$w.json; tail -3 gpurun_out/bench_$w.err
done
