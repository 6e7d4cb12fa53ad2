# multi-GPU pass: the CP tests over NCCL / peer memory (one GPU per rank), then the CP scaling
# lines (li_cp strong scaling at L = 1M, mr weak scaling) at N = 1, 2, 4
mkdir -p gpurun_out
nvidia-smi -L
timeout 1200 python -m pytest tests/test_gpu_cp.py -q -rs > gpurun_out/pytest_cp_multi.log 2>&1
echo "cp tests rc=$?"; tail -5 gpurun_out/pytest_cp_multi.log
for W in li_cp mr; do
  W=$W STEPS=${STEPS:-10} bash scripts/gpu_cp_scale.sh
done
