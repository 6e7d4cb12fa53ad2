# ncu of the fused LI mixer at the stripe's length (B=1, D=4096, L=16384, gs=1)
mkdir -p gpurun_out
cat > /tmp/li_short.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2503_01868_b200 import ops
B, D, L = 1, 4096, 16384
g = torch.Generator(device="cuda").manual_seed(0)
proj = torch.randn((B, 3 * D, L), device="cuda", generator=g).to(torch.bfloat16)
feat = (torch.randn((3, D, 7), device="cuda", generator=g) / 2.65)
packed = ops.feat_pack(feat)
res = torch.randn((D, 8), device="cuda", generator=g) / 8
poles = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
for _ in range(3):
    ops.li_mixer(proj, feat, res, poles, 1, packed=packed)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:two_stage -c 1 -o gpurun_out/li_short python /tmp/li_short.py > gpurun_out/li_short.log 2>&1
tail -2 gpurun_out/li_short.log
