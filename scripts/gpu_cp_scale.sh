# CP scaling: bench.py --workload $W at N = 1, 2, 4 on one box (each run under its own timeout)
mkdir -p gpurun_out
W=${W:-li_cp}
NG=$(nvidia-smi -L | wc -l)
for N in 1 2 4; do
  [ $N -gt $NG ] && continue
  if [ $N -eq 1 ]; then
    timeout 900 python bench.py --workload $W --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-extra-configs > gpurun_out/cp_${W}_n1.json 2> gpurun_out/cp_${W}_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 \
      bench.py --workload $W --gpus $N --steps ${STEPS:-10} --warmup 3 --no-extra-configs > gpurun_out/cp_${W}_n$N.json 2> gpurun_out/cp_${W}_n$N.err
  fi
  echo "N=$N rc=$?"; grep '^{' gpurun_out/cp_${W}_n$N.json | cut -c1-300; tail -3 gpurun_out/cp_${W}_n$N.err
done
