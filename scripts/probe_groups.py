import os, sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
from paper_2503_01868_b200 import ops
sys.path.insert(0, "scripts")
from bench_kernels import timeit, report
g = torch.Generator(device="cuda").manual_seed(0)
D = 4096
for L in (16384, 131072):
    v = torch.randn((1, D, L), device="cuda", dtype=torch.bfloat16, generator=g)
    for gs in (1, 16):
        res = torch.randn((D // gs, 8), device="cuda", generator=g) / 8
        poles = torch.rand((D // gs, 8), device="cuda", generator=g) * 1.9 - 0.95
        ms = timeit(lambda: ops.li_conv(v, res, poles, gs))
        report(f"li_conv_L{L}_gs{gs}", ms, 4 * D * L)
    proj = torch.randn((1, 3 * D, L), device="cuda", dtype=torch.bfloat16, generator=g)
    feat = torch.randn((3, D, 7), device="cuda", generator=g) / 3
    packed = ops.feat_pack(feat)
    for gs in (1, 16):
        res = torch.randn((D // gs, 8), device="cuda", generator=g) / 8
        poles = torch.rand((D // gs, 8), device="cuda", generator=g) * 1.9 - 0.95
        ms = timeit(lambda: ops.li_mixer(proj, feat, res, poles, gs, packed=packed))
        report(f"li_mixer_L{L}_gs{gs}", ms, 8 * D * L)
