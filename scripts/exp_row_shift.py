"""Probe: can a tcgen05 SW128 K-major descriptor start one 128-byte row into a swizzle atom?
Runs the two-stage kernel with T1 . U_prev replaced by the U buffer read one row back
(HY_TS_SHIFT=1: base-offset field 0; =2: base offset (addr >> 7) & 7) and compares every
output chunk except each tile's first (whose row -1 is outside the buffer) with the normal run."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
B, C, L = 1, 8, 8192
v = torch.randn((B, C, L), device="cuda", generator=g).to(torch.bfloat16)
taps = torch.randn((C, 129), device="cuda", generator=g) / 11
os.environ["HY_TS_SHIFT"] = "0"
ref = ops.two_stage(v, taps, 1).float()
mask = torch.ones(L, dtype=torch.bool, device="cuda")
for t0 in range(0, L, 4096):
    mask[t0:t0 + 128] = False
for mode in ("1", "2"):
    os.environ["HY_TS_SHIFT"] = mode
    got = ops.two_stage(v, taps, 1).float()
    d = (got - ref)[..., mask].abs().max().item()
    d0 = (got - ref)[..., ~mask].abs().max().item()
    print(f"HY_TS_SHIFT={mode}: max diff (chunks >= 1) {d:.3e}, first chunks {d0:.3e}", flush=True)
os.environ["HY_TS_SHIFT"] = "0"
