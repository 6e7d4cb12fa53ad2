"""Accuracy / speed of the split-bf16 fp32 GEMM (paper_2503_01868_b200.blas) vs native fp32."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import blas

torch.backends.cuda.matmul.allow_tf32 = False
g = torch.Generator(device="cuda").manual_seed(0)
D, L = 4096, 4096
W = torch.randn((3 * D, D), device="cuda", generator=g) / 64
x = torch.randn((1, D, L), device="cuda", generator=g)
ref = torch.matmul(W.double(), x.double())
nat = torch.matmul(W, x)
Wp = blas.split3(W)
emu = blas.matmul_split3(Wp, blas.split3(x))
den = ref.abs().max().item()
print("native rel_err", ((nat.double() - ref).abs().max().item() / den))
print("split3 rel_err", ((emu.double() - ref).abs().max().item() / den))
for name, fn in (("native", lambda: torch.matmul(W, x)), ("split3", lambda: blas.matmul_split3(Wp, blas.split3(x)))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(name, f"{ms:.3f} ms", f"{2 * 3 * D * D * L / ms / 1e9:.1f} TFLOP/s")
