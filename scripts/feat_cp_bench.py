"""hy_featurize_fwd (the CP LI featurizer stream: u = fk*fv, fq) at the N=4 segment size."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops
C, m = 1024, 262144
g = torch.Generator(device="cuda").manual_seed(0)
proj = torch.randn((1, 3 * C, m), device="cuda", generator=g).to(torch.bfloat16)
ft = torch.randn((3, C, 7), device="cuda", generator=g) / 3
for _ in range(3):
    ops.featurize(proj, ft)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    ops.featurize(proj, ft)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
nb = C * m * 2 * 5
print(f"featurize C={C} m={m}: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s")
