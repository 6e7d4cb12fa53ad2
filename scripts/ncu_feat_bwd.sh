# ncu --set full of the featurizer backward inside the C2 training step
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:feat_bwd -c 1 -o gpurun_out/feat_bwd \
  python bench.py --workload mr_train --steps 1 --warmup 3 --no-cpu-baseline --no-extra-configs > gpurun_out/feat_bwd.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/feat_bwd.log
