# C2-only launch list, the grouped-filter (d_g = 16) lines, the fused-projection headline, smoke
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-configs > /dev/null 2>&1; echo "launches rc=$?"
for w in mr li; do
  timeout 600 python bench.py --workload $w --group-size 16 --steps 10 --warmup 3 --no-extra-configs \
    > gpurun_out/g16_$w.json 2> gpurun_out/g16_$w.err; echo "g16 $w rc=$?"; cut -c1-200 gpurun_out/g16_$w.json
done
timeout 600 python bench.py --workload mr_fused --steps 10 --warmup 3 --no-extra-configs \
  > gpurun_out/final_mr_fused.json 2> gpurun_out/final_mr_fused.err; echo "mr_fused rc=$?"; cut -c1-300 gpurun_out/final_mr_fused.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
