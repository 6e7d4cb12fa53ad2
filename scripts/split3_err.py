"""Error of the split-bf16 fp32 GEMM vs the K-chunk of its leading term (C1's W_qkv shape)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import blas
torch.manual_seed(0)
M, K, N = 12288, 4096, 4096
a = (torch.randn(M, K, device="cuda", dtype=torch.float64) / K ** 0.5).float()
b = torch.randn(K, N, device="cuda", dtype=torch.float64).float()
want = a.double() @ b.double()
ws = blas.split3_weight(a)
bs = blas.split3(b)
for kc in (512, 1024, 2048, 4096):
    blas._KC = kc
    got = blas.matmul_split3(ws, bs)
    err = float((got.double() - want).abs().max() / want.abs().max())
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        blas.matmul_split3(ws, bs)
    e.record()
    torch.cuda.synchronize()
    print(f"KC={kc}: rel err {err:.2e}, {s.elapsed_time(e) / 10:.3f} ms")
