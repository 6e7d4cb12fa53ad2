# LI / SE kernel checks, each command under its own timeout
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "li or LI or se or SE" -p no:cacheprovider > gpurun_out/pytest_li.log 2>&1; echo "pytest li rc=$?"
tail -15 gpurun_out/pytest_li.log
WORKLOADS="li se stripe" bash scripts/gpu_workloads.sh
