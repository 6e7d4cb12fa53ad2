mkdir -p gpurun_out
timeout 300 python scripts/trace_li.py mixer > gpurun_out/trace_li_mixer.txt 2>&1; echo "mixer rc=$?"
