mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "li or LI or implicit or cp or mixer" > gpurun_out/li_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/li_tests.log
timeout 300 python scripts/trace_li.py mixer > gpurun_out/trace_li_mixer.txt 2>&1; echo "mixer rc=$?"
timeout 300 python scripts/trace_li.py conv > gpurun_out/trace_li_conv.txt 2>&1; echo "conv rc=$?"
timeout 600 python bench.py --workload li --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/li.json 2> gpurun_out/li.err; echo "li rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/li.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline'], d['phases_ms'])"
timeout 300 python scripts/bench_kernels.py > gpurun_out/kernels.txt 2>&1; echo "kernels rc=$?"; grep -i "li" gpurun_out/kernels.txt | head
