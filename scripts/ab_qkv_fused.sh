# A/B of the C2 operator routes on one box, alternating: cuBLAS W_qkv + fused mixer (HY_QKV_FUSED=0)
# vs the hand-written projection GEMM with the featurizers in its epilogue (HY_QKV_FUSED=1)
for i in 1 2 3 4; do
  for f in 0 1; do
    HY_QKV_FUSED=$f timeout 300 python bench.py --no-cpu-baseline --no-extra-configs --steps ${STEPS:-20} --warmup 5 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused=$f', round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,3), d['clocks']['sm_mhz'], d['clocks']['reasons'], [round(k['launch_ms'],4) for k in d['roofline_kernels']])"
  done
done
