# ncu of the inner conv on the fused projections (block_conv(u, q=fq) and two_stage(u, q=fq)) at C2 size
mkdir -p gpurun_out
cat > /tmp/inner_one.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2503_01868_b200 import ops
B, D, L = 4, 4096, 8192
u = torch.randn((B, D, L), device="cuda").to(torch.bfloat16)
fq = torch.randn((B, D, L), device="cuda").to(torch.bfloat16)
taps = torch.randn((D, 128), device="cuda") / 11.3
dec = torch.linspace(0.01, 2.0, D, device="cuda")
for _ in range(2):
    ops.block_conv(u, taps, 1, q=fq, decay=dec)
    ops.two_stage(u, taps, 1, q=fq, decay=dec)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:block_conv -c 1 -o gpurun_out/bc_fqu python /tmp/inner_one.py > gpurun_out/inner_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:two_stage -c 1 -o gpurun_out/ts_fqu python /tmp/inner_one.py >> gpurun_out/inner_ncu.log 2>&1
tail -3 gpurun_out/inner_ncu.log
