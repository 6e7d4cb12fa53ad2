import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import blas
g = torch.Generator(device="cuda").manual_seed(0)
D, L = 4096, 4096
W = torch.randn((3 * D, D), device="cuda", generator=g) / 64
x = torch.randn((D, L), device="cuda", generator=g)
ref = W.double() @ x.double(); den = ref.abs().max().item()
torch.backends.cuda.matmul.allow_tf32 = False
print("native", ((W @ x).double() - ref).abs().max().item() / den)
Wp, xp = blas.split3(W), blas.split3(x)
print("split exact?", ((Wp[0].float() + Wp[1].float() + Wp[2].float()) - W).abs().max().item())
for pairs in (((1,1),(0,2),(2,0),(0,1),(1,0),(0,0)), ((2,1),(1,2),(1,1),(0,2),(2,0),(0,1),(1,0),(0,0)),
              ((0,0),(0,1),(1,0),(1,1),(0,2),(2,0))):
    out = None
    for i, j in pairs:
        t = torch.mm(Wp[i], xp[j], out_dtype=torch.float32)
        out = t if out is None else out + t
    print(len(pairs), pairs[0], ((out.double() - ref).abs().max().item() / den))
    # fp64 accumulation of the fp32 partial products
    out = None
    for i, j in pairs:
        t = torch.mm(Wp[i], xp[j], out_dtype=torch.float32).double()
        out = t if out is None else out + t
    print("  f64 sum of parts", ((out - ref).abs().max().item() / den))
# K-split: accumulate 4 chunks of K in fp32 via separate GEMMs
out = torch.zeros((3 * D, L), device="cuda", dtype=torch.float64)
for k0 in range(0, D, 512):
    for i, j in ((1,1),(0,2),(2,0),(0,1),(1,0),(0,0)):
        out += torch.mm(Wp[i][:, k0:k0+512].contiguous(), xp[j][k0:k0+512], out_dtype=torch.float32).double()
print("ksplit512 f64 sum", ((out - ref).abs().max().item() / den))
import time
for kc in (256, 512, 1024):
    def run():
        out = torch.mm(Wp[1], xp[1], out_dtype=torch.float32)
        for i, j in ((0,2),(2,0),(0,1),(1,0)):
            torch.addmm(out, Wp[i], xp[j], out_dtype=torch.float32, out=out)
        for k0 in range(0, D, kc):
            torch.addmm(out, Wp[0][:, k0:k0+kc], xp[0][k0:k0+kc], out_dtype=torch.float32, out=out)
        return out
    o = run()
    err = ((o.double() - ref).abs().max().item() / den)
    for _ in range(2): run()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): run()
    e.record(); torch.cuda.synchronize()
    print("kc", kc, "err", err, "ms", s.elapsed_time(e) / 5)
