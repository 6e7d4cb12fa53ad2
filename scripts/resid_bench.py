"""Residual add fused into the out-projection GEMM (beta = 1) vs a separate add, C4 sizes."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01868_b200 as hy

D, L = 4096, 16384
cfg = hy.make_hyena_config("MR", D, hy.make_rng(0), inner_len=128, block_size=128)
op = hy.HyenaOperator(cfg, torch.bfloat16)
x = torch.randn((1, D, L), device="cuda").to(torch.bfloat16)
mixed = torch.randn((1, D, L), device="cuda").to(torch.bfloat16)

def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n

acc = x.clone()
for rep in range(3):
    print(rep, "full fwd + add", round(t(lambda: x + op.forward(x)), 4), "full fwd acc", round(t(lambda: op.forward(x, accumulate_into=acc)), 4),
          "mm+add", round(t(lambda: x + torch.mm(op.w_out_t, mixed[0])), 4), "addmm_", round(t(lambda: acc[0].addmm_(op.w_out_t, mixed[0])), 4))
