"""StripedHyena 2 multi-hybrid stripe (BASELINE config 4: SE-MR-LI-MHA) on the device.

The reference composes Hyena layers only (hyena.py:350-406, VARIANTS = SE/MR/LI); multi-head
attention is not part of it (SPEC non-goal), so the MHA layer here has no oracle: its parity
is unpinned. It is plain library compute: cuBLAS projections and PyTorch's fused causal
scaled-dot-product attention (flash backend), used to benchmark the stripe of the paper.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn.functional as F

from .hyena import HyenaConfig, HyenaOperator


class MHALayer:
    """Causal multi-head attention on (B, D, L) activations (random init, bf16)."""

    def __init__(self, width: int, heads: int = 32, dtype=torch.bfloat16, seed: int = 0, dev=None):
        if width % heads != 0:
            raise ValueError("width must be divisible by heads")
        self.d, self.h = width, heads
        dev = dev or torch.device("cuda")
        g = torch.Generator(device="cpu").manual_seed(seed)
        s = 1.0 / math.sqrt(width)
        self.w_qkv = (torch.randn((width, 3 * width), generator=g) * s).to(dev, dtype)
        self.w_out = (torch.randn((width, width), generator=g) * s).to(dev, dtype)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        B, D, L = x.shape
        xt = x.transpose(1, 2)  # (B, L, D)
        qkv = torch.matmul(xt, self.w_qkv).view(B, L, 3, self.h, D // self.h).permute(2, 0, 3, 1, 4)
        o = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], is_causal=True)  # (B, H, L, hd)
        o = o.permute(0, 2, 1, 3).reshape(B, L, D)
        return torch.matmul(o, self.w_out).transpose(1, 2).contiguous()

    __call__ = forward


class Stripe:
    """Hyena SE -> MR -> LI -> MHA with residual connections (hyena.py:399-406 residual form)."""

    def __init__(self, cfgs, dtype=torch.bfloat16, heads: int = 32, residual: bool = True):
        for cfg in cfgs:
            if not isinstance(cfg, HyenaConfig):
                raise TypeError("stripe layers must be HyenaConfig")
        self.ops = [HyenaOperator(cfg, dtype) for cfg in cfgs]
        self.mha = MHALayer(cfgs[0].width, heads, dtype)
        self.residual = residual

    def forward(self, x: torch.Tensor, events=None) -> torch.Tensor:
        cur = x
        for i, op in enumerate(self.ops):
            ev = None if events is None else events[i]
            if self.residual:  # residual add in the out-projection GEMM epilogue
                cur = op.forward(cur, events=ev, accumulate_into=cur.clone() if i == 0 else cur)
            else:
                cur = op.forward(cur, events=ev)
        out = self.mha(cur)
        return cur + out if self.residual else out

    __call__ = forward
