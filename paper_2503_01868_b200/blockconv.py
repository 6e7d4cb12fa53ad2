"""Blocked causal convolution API (blockconv.py of the reference) over the GPU kernels.

`two_stage_forward`, `block_conv` and `chunk_parallel_forward` keep the
reference signatures, validation and exceptions; the arithmetic runs on the
device: fp32 / fp64 SeqTensors use the CUDA-core FIR kernel (exact fp32 / fp64
accumulation of the same causal sum), bf16 device tensors use the tcgen05
two-stage kernel (ops.two_stage). The factor helpers (build_factors,
assemble_toeplitz) are host-side utilities, as in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .core import GroupSpec, SeqTensor, device, from_device, group_taps_device, to_device


class TwoStageIneligibleError(ValueError):
    """Filter needs more than one spill factor; route to block_conv instead (blockconv.py:27-28)."""


@dataclass
class MultiplyCounter:
    """Tallies scalar multiplies of the dense two-factor model (blockconv.py:31-38)."""

    multiplies: int = 0

    def add_matmul(self, m: int, k: int, n: int) -> None:
        self.multiplies += m * k * n


@dataclass(frozen=True)
class ToeplitzFactors:
    blocks: np.ndarray  # (spill_count + 1, block_size, block_size)
    block_size: int
    filter_len: int

    @property
    def spill_count(self) -> int:
        return self.blocks.shape[0] - 1


def spill_count(filter_len: int, block_size: int) -> int:
    """ceil((filter_len - 1) / block_size) (blockconv.py:54-56)."""
    return math.ceil((filter_len - 1) / block_size)


def build_factors(taps, block_size: int) -> ToeplitzFactors:
    """B_k[i, j] = h[k*lb + i - j] masked to [0, lh) (blockconv.py:59-74). Host utility; the
    tcgen05 kernel builds the same T0/T1 in shared memory from the taps."""
    taps = np.asarray(taps, dtype=np.float64)
    if taps.ndim != 1 or taps.size < 1:
        raise ValueError("need a nonempty 1-d tap vector")
    if block_size < 1:
        raise ValueError(f"block_size must be >= 1, got {block_size}")
    lh = taps.size
    k_count = spill_count(lh, block_size)
    lag = (np.arange(k_count + 1)[:, None, None] * block_size + np.arange(block_size)[None, :, None]
           - np.arange(block_size)[None, None, :])
    valid = (lag >= 0) & (lag < lh)
    blocks = np.where(valid, taps[np.clip(lag, 0, lh - 1)], 0.0)
    return ToeplitzFactors(blocks, block_size, lh)


def assemble_toeplitz(factors: ToeplitzFactors, length: int) -> np.ndarray:
    """Factors laid on block diagonals = dense Toeplitz (blockconv.py:77-86). Host utility."""
    lb = factors.block_size
    n = math.ceil(length / lb)
    full = np.zeros((n * lb, n * lb))
    for row in range(n):
        for k in range(min(row, factors.spill_count) + 1):
            col = row - k
            full[row * lb:(row + 1) * lb, col * lb:(col + 1) * lb] = factors.blocks[k]
    return full[:length, :length]


def _require_two_stage(filter_len: int, block_size: int) -> None:
    if spill_count(filter_len, block_size) > 1:
        raise TwoStageIneligibleError(
            f"filter_len {filter_len} needs {spill_count(filter_len, block_size)} spill factors "
            f"at block_size {block_size}; the two-stage kernel holds one — use block_conv")


def block_conv(x: SeqTensor, groups: GroupSpec, block_size: int) -> SeqTensor:
    """General blocked conv, any filter length (blockconv.py:103-121); same causal sum on the GPU."""
    from .ops import causal_conv
    if x.channels != groups.channels:
        raise ValueError(f"input has {x.channels} channels, grouping expects {groups.channels}")
    if block_size < 1:
        raise ValueError(f"block_size must be >= 1, got {block_size}")
    xd = to_device(x)
    y = causal_conv(xd, group_taps_device(groups, xd.dtype), groups.group_size)
    return from_device(y, x.dtype)


@dataclass
class TwoStageSaved:
    """Forward context (blockconv.py:139-149); arrays are host copies."""

    v: SeqTensor
    q: SeqTensor | None
    k: SeqTensor | None
    groups: GroupSpec
    block_size: int
    gated_input: np.ndarray
    conv_out: np.ndarray


def _check_two_stage(v, groups, block_size, q, k):
    if v.channels != groups.channels:
        raise ValueError(f"input has {v.channels} channels, grouping expects {groups.channels}")
    for name, gate in (("q", q), ("k", k)):
        if gate is not None and (gate.channels, gate.length) != (v.channels, v.length):
            raise ValueError(f"gate {name} shape {(gate.channels, gate.length)} "
                             f"does not match input {(v.channels, v.length)}")
    _require_two_stage(groups.filter_len, block_size)


def _count(counter, groups, block_size, length):
    if counter is not None:
        n = math.ceil(length / block_size)
        for _ in range(groups.n_groups):
            counter.add_matmul(block_size, block_size, groups.group_size * n)
            counter.add_matmul(block_size, block_size, groups.group_size * n)


def two_stage_forward(v: SeqTensor, groups: GroupSpec, block_size: int, q: SeqTensor | None = None,
                      k: SeqTensor | None = None, counter: MultiplyCounter | None = None) -> SeqTensor:
    """y = q * conv(k * v), requires filter_len <= block_size + 1 (blockconv.py:182-220)."""
    from .ops import gated_conv
    _check_two_stage(v, groups, block_size, q, k)
    _count(counter, groups, block_size, v.length)
    vd = to_device(v)
    qd = None if q is None else to_device(SeqTensor(q.data, dtype=v.dtype))
    kd = None if k is None else to_device(SeqTensor(k.data, dtype=v.dtype))
    y = gated_conv(vd, group_taps_device(groups, vd.dtype), groups.group_size, q=qd, k=kd)
    return from_device(y, v.dtype)


def two_stage_forward_saved(v: SeqTensor, groups: GroupSpec, block_size: int, q: SeqTensor | None = None,
                            k: SeqTensor | None = None, counter: MultiplyCounter | None = None):
    """Forward half of blockconv.py:199-220: (y, TwoStageSaved)."""
    import torch

    from .ops import gated_conv
    _check_two_stage(v, groups, block_size, q, k)
    _count(counter, groups, block_size, v.length)
    vd = to_device(v).to(torch.float64)
    u = vd * to_device(k).to(torch.float64) if k is not None else vd
    c = gated_conv(u, group_taps_device(groups, torch.float64), groups.group_size)
    y = c * to_device(q).to(torch.float64) if q is not None else c
    saved = TwoStageSaved(v, q, k, groups, block_size, u.cpu().numpy(), c.cpu().numpy())
    return SeqTensor(y.cpu().numpy(), dtype=v.dtype), saved


@dataclass
class TwoStageGrads:
    """(blockconv.py:152-157)."""

    dv: np.ndarray
    dq: np.ndarray | None
    dk: np.ndarray | None
    dtaps: np.ndarray  # (n_groups, filter_len)


def two_stage_backward(saved: TwoStageSaved, dy) -> TwoStageGrads:
    """Analytic gradients of the gated two-stage forward (blockconv.py:223-264) on the GPU, fp64:
    dq = dy * conv_out, dc = dy * q, du = the transposed-factor (anti-causal) conv of dc, and the
    filter gradient by the deterministic two-pass correlation (per-CTA partials, fixed-order
    reduce) of hy_causal_conv_bwd; dk = du * v, dv = du * k."""
    import torch

    from .ops import causal_conv_bwd
    if not isinstance(saved, TwoStageSaved):
        raise ValueError("backward needs the TwoStageSaved context from two_stage_forward_saved")
    dy = dy.data if isinstance(dy, SeqTensor) else np.asarray(dy, dtype=np.float64)
    if dy.shape != saved.gated_input.shape:
        raise ValueError(f"dy shape {dy.shape} does not match forward shape {saved.gated_input.shape}")
    dev = device()
    f64 = lambda a: torch.from_numpy(np.array(a, dtype=np.float64, copy=True)).to(dev)  # noqa: E731
    dyd = f64(dy)
    qd = None if saved.q is None else f64(saved.q.data)
    dq = dyd * f64(saved.conv_out) if qd is not None else None
    dc = dyd * qd if qd is not None else dyd
    groups = saved.groups
    du, dtaps = causal_conv_bwd(dc, f64(saved.gated_input), group_taps_device(groups, torch.float64),
                                groups.group_size)
    dk = du * f64(saved.v.data) if saved.k is not None else None
    dv = du * f64(saved.k.data) if saved.k is not None else du
    h = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
    return TwoStageGrads(dv=h(dv), dq=h(dq), dk=h(dk), dtaps=h(dtaps))


def chunk_parallel_forward(v: SeqTensor, taps, block_size: int, counter: MultiplyCounter | None = None) -> SeqTensor:
    """One shared tap vector for every channel (blockconv.py:267-293)."""
    import torch

    from .ops import causal_conv, tap_dtype
    taps = np.asarray(taps, dtype=np.float64)
    _require_two_stage(taps.size, block_size)
    if counter is not None:
        n = math.ceil(v.length / block_size)
        counter.add_matmul(block_size, block_size, n * v.channels)
        counter.add_matmul(block_size, block_size, n * v.channels)
    vd = to_device(v)
    t = torch.from_numpy(taps[None, :]).to(device(), dtype=tap_dtype(vd.dtype))
    return from_device(causal_conv(vd, t, v.channels), v.dtype)


def two_stage_flops(length: int, block_size: int, channels: int) -> int:
    """Multiply count of the dense two-factor path: 2 * lb^2 * d * ceil(l/lb) (blockconv.py:296-300)."""
    if length < 1 or block_size < 1 or channels < 1:
        raise ValueError("length, block_size, and channels must all be >= 1")
    return 2 * block_size * block_size * channels * math.ceil(length / block_size)
