# Round-1 CP evidence on a 4-GPU box: the multi-GPU tests, then LI and MR CP scaling at N = 1, 2, 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu4.log
W=li_cp bash scripts/gpu_cp_scale.sh
W=mr bash scripts/gpu_cp_scale.sh
