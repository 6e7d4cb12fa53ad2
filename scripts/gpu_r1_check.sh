# Round-1 check after host-side launcher changes: GPU tests, smoke, default bench, kernel timings
mkdir -p gpurun_out
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke2.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu2.log
timeout 900 python scripts/bench_kernels.py --which se > gpurun_out/kernels_se.jsonl 2>&1; echo "bk rc=$?"; cut -c1-200 gpurun_out/kernels_se.jsonl
timeout 900 python scripts/bench_kernels.py --which li > gpurun_out/kernels_li.jsonl 2>&1; cut -c1-200 gpurun_out/kernels_li.jsonl
timeout 900 python scripts/bench_kernels.py --which mr > gpurun_out/kernels_mr.jsonl 2>&1; cut -c1-200 gpurun_out/kernels_mr.jsonl
for W in mr se; do timeout 900 python bench.py --workload $W > gpurun_out/bench2_$W.json 2> gpurun_out/bench2_$W.err; echo "bench $W rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/bench2_$W.json').read().strip().splitlines()[-1]); print('$W', d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"; done
