import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2503_01868_b200 import ops
D, L = 512, 131072
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.randn((1, D, L), device="cuda", dtype=torch.bfloat16, generator=g)
taps = torch.randn((D, L), device="cuda", generator=g) / 100
ops.fft_conv(v, taps, 1, q=v, k=v)
torch.cuda.synchronize()
