mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_cp.py -q --timeout 600 -p no:cacheprovider > gpurun_out/cp_tests.log 2>&1; echo "cp tests rc=$?"; tail -3 gpurun_out/cp_tests.log
for N in 2 4; do
  for S in serial concurrent; do
    HY_CP_LI_SCHED=$S timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29617 \
      bench.py --workload li_cp --gpus $N --steps 5 --warmup 3 > gpurun_out/licp_n${N}_$S.json 2> gpurun_out/licp_n${N}_$S.err
    echo "N=$N $S rc=$?"; python -c "import json; d=json.loads([l for l in open('gpurun_out/licp_n${N}_$S.json') if l.startswith('{')][-1]); print(round(d['ms_per_step'],2), d['phases_ms'], d['clocks']['sm_mhz'])"
  done
done
