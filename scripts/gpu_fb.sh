mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_backward_kernels.py -q --timeout 300 -p no:cacheprovider > gpurun_out/bwd_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bwd_tests.log
timeout 600 python scripts/bench_backward.py > gpurun_out/bk_bwd.txt 2>&1; echo "bk rc=$?"; cat gpurun_out/bk_bwd.txt | head -20
timeout 600 python bench.py --workload mr_train --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/mrt.json 2> gpurun_out/mrt.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/mrt.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_ms'], d['phases_ms'])"
