mkdir -p gpurun_out
for P in 8 2; do
  HY_CP_NPIPE=$P timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29619 \
    bench.py --workload li_cp --gpus 4 --steps 5 --warmup 3 > gpurun_out/licp_n4_p$P.json 2> gpurun_out/licp_n4_p$P.err
  echo "N=4 npipe=$P rc=$?"; python -c "import json; d=json.loads([l for l in open('gpurun_out/licp_n4_p$P.json') if l.startswith('{')][-1]); print(round(d['ms_per_step'],2), d['phases_ms'], d['clocks']['sm_mhz'])"
done
