# GPU pass: every -m gpu test (no -x: see all failures), then the default bench line
mkdir -p gpurun_out
nvidia-smi -L
timeout ${PT_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rs --durations=20 ${PT_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -40 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; cut -c1-3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
