"""Kernel F (standalone featurizer, hy_causal_conv_fwd) at SURVEY 7.3's size: 3*4096 rows x 4096, fp32, lh 7."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn((1, 3 * 4096, 4096), device="cuda", generator=g)
taps = torch.randn((3 * 4096, 7), device="cuda", generator=g) / 3
for _ in range(3):
    ops.causal_conv(x, taps, 1)
torch.cuda.synchronize()
