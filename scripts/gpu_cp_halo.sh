# MR CP halo over peer copies vs NCCL: CP tests, then the MR CP bench at N=1 and N=2 (20 steps)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cp.py -q --timeout 600 -p no:cacheprovider > gpurun_out/cp_tests.log 2>&1; echo "cp tests rc=$?"; tail -3 gpurun_out/cp_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mr_n1.json 2> gpurun_out/mr_n1.err; echo "n1 rc=$?"
for P in 1 0; do
  HY_CP_P2P=$P timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 \
    bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/mr_n2_p$P.json 2> gpurun_out/mr_n2_p$P.err; echo "n2 p2p=$P rc=$?"; tail -2 gpurun_out/mr_n2_p$P.err
done
for f in mr_n1 mr_n2_p1 mr_n2_p0; do python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/$f.json') if l.startswith('{')][-1]); print('$f', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,2), 'Mtok/s', d['phases_ms'])"; done
