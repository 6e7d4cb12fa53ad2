mkdir -p gpurun_out
cat > /tmp/qg_one.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2503_01868_b200 import ops
B, D, L = 4, 4096, 8192
x = torch.randn((B, D, L), device="cuda").to(torch.bfloat16)
w = (torch.randn((3 * D, D), device="cuda") / 64).to(torch.bfloat16)
feat = torch.randn((3, D, 7), device="cuda") / 2.65
wp = ops.qkv_weight_permute(w)
for _ in range(2):
    ops.qkv_feat_gemm(x, wp, feat)
torch.matmul(w, x)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:qkv_feat_gemm -c 1 -o gpurun_out/qg3_full python /tmp/qg_one.py > gpurun_out/qg_ncu.log 2>&1

tail -5 gpurun_out/qg_ncu.log
