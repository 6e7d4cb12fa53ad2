"""MHA layer of the stripe (C4: L=16384, D=4096, 32 heads) under each SDPA backend."""
import os, sys
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200.stripe import MHALayer

L, D, H = 16384, 4096, 32
mha = MHALayer(D, H)
x = torch.randn((1, D, L), device="cuda").to(torch.bfloat16)
q = torch.randn((1, H, L, D // H), device="cuda").to(torch.bfloat16)

def t(fn, n=10):
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

print("layer default", t(lambda: mha(x)))
for be in (SDPBackend.FLASH_ATTENTION, SDPBackend.CUDNN_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
    try:
        with sdpa_kernel([be]):
            ms = t(lambda: F.scaled_dot_product_attention(q, q, q, is_causal=True))
            ml = t(lambda: mha(x))
        print(be, "attn", round(ms, 3), "ms", round(2 * L * L * D / ms / 1e9, 1), "TF/s; layer", round(ml, 3))
    except Exception as e:
        print(be, "failed", str(e)[:200])
