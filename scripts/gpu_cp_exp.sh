# li_cp at N=2, 4: NVLink peer-memory all-to-all vs NCCL, two pipeline depths
mkdir -p gpurun_out
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29612 \
      bench.py --workload li_cp --gpus $2 --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/exp_$1.err | grep '^{' | tee gpurun_out/exp_$1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2))"; }
timeout 900 python -m pytest tests/test_gpu_cp.py -q --timeout 600 -p no:cacheprovider 2>&1 | tail -2
HY_CP_NPIPE=4 run p2p_np4_n4 4
HY_CP_NPIPE=8 run p2p_np8_n4 4
HY_CP_P2P=0 HY_CP_NPIPE=8 run nccl_np8_n4 4
HY_CP_NPIPE=4 run p2p_np4_n2 2
HY_CP_NPIPE=8 run p2p_np8_n2 2
