"""FFT-conv API of the reference (fft.py) on the GPU.

`fft_conv(x, taps)` keeps the reference contract (fft.py:128-145): causal FIR of
the last axis, zero padded so there is no wraparound, float64 result.
"""

from __future__ import annotations

import numpy as np
import torch


def require_pow2(n: int) -> int:
    if n < 1 or (n & (n - 1)) != 0:
        raise ValueError(f"length must be a power of two, got {n}")
    return n


def next_pow2(n: int) -> int:
    """Smallest power of two >= n (fft.py:30-34)."""
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    return 1 << (n - 1).bit_length()


def fft_conv(x, taps) -> np.ndarray:
    """Causal conv of the last axis with per-row or shared taps; float64 (fft.py:128-145).

    Runs on the device in fp64 through ops.long_conv (FFT kernel when built,
    the fp64 FIR kernel otherwise) — same numbers as the zero-padded transform.
    """
    from .core import device
    from .ops import long_conv
    x = np.asarray(x, dtype=np.float64)
    taps = np.asarray(taps, dtype=np.float64)
    l = x.shape[-1]
    rows = x.reshape(-1, l)
    xd = torch.from_numpy(np.ascontiguousarray(rows)).to(device())
    if taps.ndim == 1:
        td = torch.from_numpy(taps[None, :].copy()).to(device())
        gs = rows.shape[0]
    else:
        if taps.shape[:-1] != x.shape[:-1]:
            raise ValueError(f"taps leading shape {taps.shape[:-1]} does not match input {x.shape[:-1]}")
        td = torch.from_numpy(np.ascontiguousarray(taps.reshape(-1, taps.shape[-1]))).to(device())
        gs = 1
    y = long_conv(xd, td, gs)
    return y.cpu().numpy().reshape(x.shape)
