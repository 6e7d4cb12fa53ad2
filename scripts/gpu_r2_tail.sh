# end-of-round refresh: kernel micro-benchmarks and an ncu capture of the fp32 modal-scan mixer
mkdir -p gpurun_out
timeout 900 python scripts/bench_kernels.py > gpurun_out/tail_kernels.jsonl 2> gpurun_out/tail_kernels.err; echo "kernels rc=$?"
cat > /tmp/lis_one.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2503_01868_b200 import ops
D, L = 4096, 131072
g = torch.Generator(device="cuda").manual_seed(0)
proj = torch.randn((1, 3 * D, L), device="cuda", generator=g)
feat = torch.randn((3, D, 7), device="cuda", generator=g) / 2.65
res = (torch.randn((D, 8), device="cuda", generator=g) / 8).double()
poles = (torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95).double()
for _ in range(2):
    ops.li_scan_mixer(proj, feat, res, poles, 1)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:li_scan_kernel -c 1 -o gpurun_out/lis_f32 python /tmp/lis_one.py > gpurun_out/lis_ncu.log 2>&1; echo "ncu rc=$?"
