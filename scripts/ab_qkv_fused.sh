mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --no-extra-configs --steps 40 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['ms_per_step'], d['clocks']['sm_mhz'], d['e2e']['value'])"
  HY_QKV_FUSED=1 timeout 300 python bench.py --no-cpu-baseline --no-extra-configs --steps 40 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused  ', d['ms_per_step'], d['clocks']['sm_mhz'], d['e2e']['value'])"
done
