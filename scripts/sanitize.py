"""compute-sanitizer driver (racecheck / synccheck) for the mbarrier-pipelined tcgen05 kernels at
multi-group sizes: every CTA walks several tiles and filter groups (T0 double buffer, T1 rebuild,
ring phase wraps), as in the C2 / C3 benchmarks. Run under
    compute-sanitizer --tool racecheck python scripts/sanitize.py <case>
One launch per case (sanitizer tools replay slowly)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops  # noqa: E402

case = sys.argv[1]
g = torch.Generator(device="cuda").manual_seed(0)
C, L = 512, 8192  # 4 tiles per sequence (32-chunk kernel); ~28 tiles and 7 groups per CTA
if case == "mr_mixer":  # two_stage_kernel<FEAT>
    proj = torch.randn((1, 3 * C, L), device="cuda", generator=g).to(torch.bfloat16)
    feat = torch.randn((3, C, 7), device="cuda", generator=g) / 3
    taps = torch.randn((C, 128), device="cuda", generator=g) / 11
    ops.hyena_mixer(proj, feat, taps, 1, decay=torch.linspace(0.01, 2.0, C, device="cuda"))
elif case == "li_mixer":  # two_stage_kernel<FEAT, IMPL>
    proj = torch.randn((1, 3 * C, L), device="cuda", generator=g).to(torch.bfloat16)
    feat = torch.randn((3, C, 7), device="cuda", generator=g) / 3
    res = torch.randn((C, 8), device="cuda", generator=g) / 8
    poles = torch.rand((C, 8), device="cuda", generator=g) * 1.9 - 0.95
    ops.li_mixer(proj, feat, res, poles, 1)
elif case == "li_conv":  # block_conv_kernel<IMPL> (gated)
    v, q, k = (torch.randn((1, C, 4 * L), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    res = torch.randn((C, 8), device="cuda", generator=g) / 8
    poles = torch.rand((C, 8), device="cuda", generator=g) * 1.9 - 0.95
    ops.li_conv(v, res, poles, 1, q=q, k=k)
elif case == "block_conv":  # block_conv_kernel explicit, K = 3, gated, decay
    v, q, k = (torch.randn((1, C, 2 * L), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    taps = torch.randn((C, 385), device="cuda", generator=g) / 20
    ops.block_conv(v, taps, 1, q=q, k=k, decay=torch.linspace(0.001, 0.01, C, device="cuda"))
elif case == "taps_grad":  # taps_grad_kernel
    dc, u = (torch.randn((2, C, L), device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    ops.two_stage_taps_grad(dc, u, 128, 1)
torch.cuda.synchronize()
print("sanitize case done:", case)
