# compute-sanitizer racecheck + synccheck on the tcgen05 pipelines (summaries -> gpurun_out/)
mkdir -p gpurun_out
for c in ${CASES:-mr_mixer li_mixer li_conv block_conv taps_grad}; do
  for tool in racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py $c > gpurun_out/san_${tool}_$c.log 2>&1
    echo "$tool $c rc=$?"; tail -3 gpurun_out/san_${tool}_$c.log
  done
done
