import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops
g = torch.Generator(device="cuda").manual_seed(0)
D, L = 4096, 131072
dc = torch.randn((1, D, L), device="cuda", dtype=torch.bfloat16, generator=g)
u = torch.randn((1, D, L), device="cuda", dtype=torch.bfloat16, generator=g)
r = torch.randn((D, 8), device="cuda", generator=g) / 8
p = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
for _ in range(3):
    ops.li_param_grad(dc, u, r, p, 1)
torch.cuda.synchronize()
