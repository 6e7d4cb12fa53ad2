"""The reference's fft module (fft.py) on the GPU.

`fft_conv(x, taps)` keeps the reference contract (fft.py:128-145): causal FIR of the last
axis, zero padded so there is no wraparound, float64 result (through ops.long_conv). The
transform building blocks keep their reference names and semantics (last axis, power-of-two
lengths, complex128, `fft` unnormalised, `ifft` carrying 1/l) and run on the device: the
standalone transforms through the hand-written Stockham kernel (csrc/fft_c2c.cu), the radix-2
stages, permutations and O(l^2) oracles as device tensor ops. Results come back as numpy
arrays like the reference's.
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
    taps = taps[..., :l]  # lags >= l never reach the l outputs (same numbers as the padded transform)
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


def _dev(a, dtype=torch.complex128) -> torch.Tensor:
    from .core import device
    return torch.as_tensor(np.asarray(a)).to(device(), dtype)


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def bit_reversal_indices(l: int) -> np.ndarray:
    """(fft.py:55-63)"""
    require_pow2(l)
    bits = l.bit_length() - 1
    idx = np.arange(l)
    rev = np.zeros(l, dtype=np.int64)
    for _ in range(bits):
        rev = (rev << 1) | (idx & 1)
        idx >>= 1
    return rev


def bit_reversal(x) -> np.ndarray:
    """Permute the last axis into bit-reversed order (fft.py:66-69), on the device."""
    from .core import device
    x = np.asarray(x)
    t = torch.as_tensor(x).to(device())
    idx = torch.as_tensor(bit_reversal_indices(x.shape[-1]), device=t.device)
    return _host(t.index_select(-1, idx))


def _phase(l: int, sign: float, dev) -> torch.Tensor:
    jk = (torch.arange(l, device=dev, dtype=torch.int64)[:, None] *
          torch.arange(l, device=dev, dtype=torch.int64)[None, :]) % l
    ang = sign * 2.0 * np.pi * jk.to(torch.float64) / l
    return torch.polar(torch.ones_like(ang), ang)


def dft_oracle(x) -> np.ndarray:
    """Literal O(l^2) DFT, y[k] = sum_j x[j] exp(-2 pi i j k / l) (fft.py:37-43)."""
    t = _dev(x)
    return _host(t @ _phase(t.shape[-1], -1.0, t.device))


def idft_oracle(y) -> np.ndarray:
    """Literal inverse with 1/l (fft.py:46-52)."""
    t = _dev(y)
    return _host((t @ _phase(t.shape[-1], 1.0, t.device)) / t.shape[-1])


def dif_split(x) -> tuple:
    """One decimation-in-frequency stage (fft.py:72-85): (lo + hi, (lo - hi) W)."""
    t = _dev(x)
    l = require_pow2(t.shape[-1])
    if l < 2:
        raise ValueError("need length >= 2 to split")
    half = l // 2
    lo, hi = t[..., :half], t[..., half:]
    ang = -2.0 * np.pi * torch.arange(half, device=t.device, dtype=torch.float64) / l
    w = torch.polar(torch.ones_like(ang), ang)
    return _host(lo + hi), _host((lo - hi) * w)


def dit_merge(a, b) -> np.ndarray:
    """Inverse of dif_split with conjugate twiddles and 1/2 (fft.py:88-97)."""
    ta, tb = _dev(a), _dev(b)
    if ta.shape != tb.shape:
        raise ValueError(f"halves must match, got {tuple(ta.shape)} and {tuple(tb.shape)}")
    half = ta.shape[-1]
    ang = 2.0 * np.pi * torch.arange(half, device=ta.device, dtype=torch.float64) / (2 * half)
    bw = tb * torch.polar(torch.ones_like(ang), ang)
    return _host(torch.cat([0.5 * (ta + bw), 0.5 * (ta - bw)], dim=-1))


def _dif_passes(x) -> np.ndarray:
    """All DiF stages: natural-order input -> bit-reversed spectrum (fft.py:100-113)."""
    z = _dev(x).clone()
    l = require_pow2(z.shape[-1])
    span = l // 2
    while span >= 1:
        blocks = z.reshape(z.shape[:-1] + (-1, 2, span))
        lo = blocks[..., 0, :].clone()
        hi = blocks[..., 1, :].clone()
        ang = -2.0 * np.pi * torch.arange(span, device=z.device, dtype=torch.float64) / (2 * span)
        w = torch.polar(torch.ones_like(ang), ang)
        blocks[..., 0, :] = lo + hi
        blocks[..., 1, :] = (lo - hi) * w
        span //= 2
    return _host(z)


def fft(x) -> np.ndarray:
    """Natural-order FFT of the last axis, power-of-two length, no scale (fft.py:116-118), by the
    hand-written Stockham kernel (hy_fft_c2c)."""
    from .ops import fft_c2c
    t = _dev(x)
    require_pow2(t.shape[-1])
    return _host(fft_c2c(t))


def ifft(y) -> np.ndarray:
    """Inverse transform carrying the full 1/l (fft.py:121-125) (hy_fft_c2c)."""
    from .ops import fft_c2c
    t = _dev(y)
    require_pow2(t.shape[-1])
    return _host(fft_c2c(t, inverse=True))


def circular_conv_oracle(x, h) -> np.ndarray:
    """Literal circular convolution y[t] = sum_k h[(t - k) mod l] x[k] (fft.py:148-157)."""
    x = np.asarray(x)
    h = np.asarray(h)
    l = x.shape[-1]
    if h.shape[-1] != l:
        raise ValueError(f"signal and filter lengths differ: {l} vs {h.shape[-1]}")
    cplx = np.iscomplexobj(x) or np.iscomplexobj(h)
    dt = torch.complex128 if cplx else torch.float64
    tx, th = _dev(x, dt), _dev(h, dt)
    lag = (torch.arange(l, device=tx.device)[:, None] - torch.arange(l, device=tx.device)[None, :]) % l
    return _host(torch.einsum("...tk,...k->...t", th[..., lag], tx))
