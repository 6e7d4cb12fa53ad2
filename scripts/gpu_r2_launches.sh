# ncu launch lists (kernel shares of each workload's step) + fresh li bench line
mkdir -p gpurun_out
for w in stripe li se li_f32; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches $w rc=$?"
done
timeout 900 python bench.py --workload li --steps 10 --warmup 3 > gpurun_out/final_li.json 2> gpurun_out/final_li.err; echo "li rc=$?"
timeout 900 python scripts/bench_kernels.py --which scan > gpurun_out/kern_scan.jsonl 2>&1; echo "scan rc=$?"
