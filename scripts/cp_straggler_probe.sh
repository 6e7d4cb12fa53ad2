# N=4 default bench repeated: per-rank step times (a straggler rank shows up here)
mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 2963$i bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/strag_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/strag_$i.json')); print('run $i', round(d['ms_per_step'],3), [round(v,3) for v in d['ms_per_step_per_rank']], 'li_cp', round(d['other_configs']['li_cp']['ms_per_step'],2))"
done
