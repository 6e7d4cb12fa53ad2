"""Gated convolution operators (Hyena-SE / MR / LI) and multi-hybrid stacks on B200.

Mirrors /root/reference/pkg/src/convhybrid/hyena.py: HyenaConfig, hyena_forward,
LayoutSpec / OperatorStack / build_layout / layout_forward and the seeded
builders keep their names, arguments, validation and errors. The forward runs
on the device:

    proj  = W_qkv^T x                 cuBLAS GEMM, (B, 3D, L)    (hyena.py:124 x3, fused)
    mixed = q * inner(k * v)          one fused sm_100a kernel    (hyena.py:125, 170-186)
    y     = W_out^T mixed             cuBLAS GEMM                 (hyena.py:188)

`HyenaOperator` is the torch-native entry ((B, D, L) device tensors, parameters
packed once on the device); `hyena_forward` stages a SeqTensor through it.
"""

from __future__ import annotations

import os
import weakref
from dataclasses import dataclass
from typing import Union

import numpy as np
import torch

from . import blas, ops
from .blockconv import spill_count
from .core import (
    ExplicitFilter,
    GroupSpec,
    ImplicitFilter,
    RegularizedFilter,
    SeqTensor,
    device,
    from_device,
    to_device,
)

VARIANTS = ("SE", "MR", "LI")
LI_SCAN_MAX_POLES = 64  # hy_li_scan_fwd
BACKENDS = ("direct", "blocked", "fft")
MAX_SHORT_FILTER = 14

Projection = Union[np.ndarray, tuple]


def _as_projection(p, width: int, name: str) -> Projection:
    if isinstance(p, tuple):
        if len(p) != 2:
            raise ValueError(f"factored projection {name} must be a (left, right) pair")
        left = np.asarray(p[0], dtype=np.float64)
        right = np.asarray(p[1], dtype=np.float64)
        if left.ndim != 2 or right.ndim != 2 or left.shape[0] != width or right.shape[1] != width \
                or left.shape[1] != right.shape[0]:
            raise ValueError(f"factored projection {name} needs shapes (d, r), (r, d) with d={width}")
        return (left, right)
    arr = np.asarray(p, dtype=np.float64)
    if arr.shape != (width, width):
        raise ValueError(f"projection {name} must be ({width}, {width}), got {arr.shape}")
    return arr


def projection_dense(p: Projection) -> np.ndarray:
    """(hyena.py:64-65); factored projections are densified once at packing time."""
    return p[0] @ p[1] if isinstance(p, tuple) else p


def _check_feat(groups: GroupSpec, width: int, name: str) -> None:
    if groups.channels != width:
        raise ValueError(f"{name} covers {groups.channels} channels, operator width is {width}")
    for f in groups.filters:
        if not isinstance(f, ExplicitFilter):
            raise ValueError(f"{name} filters must be explicit short taps")
    if groups.filter_len > MAX_SHORT_FILTER:
        raise ValueError(f"{name} filter length {groups.filter_len} exceeds short-filter cap {MAX_SHORT_FILTER}")


_INNER_KIND = {"SE": ExplicitFilter, "MR": RegularizedFilter, "LI": ImplicitFilter}


@dataclass(frozen=True, eq=False)
class HyenaConfig:
    """One operator instance (hyena.py:81-119)."""

    variant: str
    width: int
    w_q: Projection
    w_k: Projection
    w_v: Projection
    w_out: Projection
    q_feat: GroupSpec
    k_feat: GroupSpec
    v_feat: GroupSpec
    inner: GroupSpec
    block_size: int = 16
    backend: str = "blocked"

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}, got {self.variant!r}")
        if self.backend not in BACKENDS:
            raise ValueError(f"backend must be one of {BACKENDS}, got {self.backend!r}")
        if self.width < 1:
            raise ValueError("width must be >= 1")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        for name in ("w_q", "w_k", "w_v", "w_out"):
            object.__setattr__(self, name, _as_projection(getattr(self, name), self.width, name))
        for name in ("q_feat", "k_feat", "v_feat"):
            _check_feat(getattr(self, name), self.width, name)
        if self.inner.channels != self.width:
            raise ValueError(f"inner filters cover {self.inner.channels} channels, width is {self.width}")
        kind = _INNER_KIND[self.variant]
        for f in self.inner.filters:
            if not isinstance(f, kind):
                raise ValueError(f"variant {self.variant} requires {kind.__name__} inner filters, "
                                 f"got {type(f).__name__}")
        if self.variant == "SE" and self.inner.filter_len > MAX_SHORT_FILTER:
            raise ValueError(f"SE inner filter length {self.inner.filter_len} exceeds {MAX_SHORT_FILTER}")


# ---------------------------------------------------------------- device operator


def _implicit_taps_device(inner: GroupSpec, dev, dtype) -> torch.Tensor:
    """h_t = sum_n R_n lambda_n^t (core.py:147-151) evaluated on the device in fp64."""
    res = torch.from_numpy(np.stack([f.residues for f in inner.filters])).to(dev)
    poles = torch.from_numpy(np.stack([f.poles for f in inner.filters])).to(dev)
    L = inner.filter_len
    out = torch.empty((inner.n_groups, L), dtype=torch.float64, device=dev)
    step = 8192
    for s in range(0, L, step):
        t = torch.arange(s, min(L, s + step), dtype=torch.float64, device=dev)
        # poles**t with 0**0 = 1, as numpy
        pw = torch.pow(poles[:, None, :], t[None, :, None])
        out[:, s:s + t.numel()] = (pw * res[:, None, :]).sum(-1)
    return out.to(dtype)


def fused_mixer_eligible(dtype: torch.dtype, lh: int, L: int) -> bool:
    """The routing rule of hy_hyena_mixer_fwd (csrc/mixer.cu): the tcgen05 mixer for bf16 with
    lh <= 129 on rows of L % 8 == 0, else the CUDA-core SE stream mixer for lh <= 16 (fp32 /
    bf16, any L). Anything else composes the unfused kernels."""
    if dtype == torch.bfloat16 and lh <= 129 and L % 8 == 0:
        return True
    return dtype in (torch.float32, torch.bfloat16) and lh <= 16


class HyenaOperator:
    """Device-resident parameters of one HyenaConfig and the torch-native forward.

    forward(x) takes a contiguous CUDA tensor (B, D, L) (or (D, L)) of the
    operator's dtype (float32, bfloat16 or float64) and returns y of the same
    shape: two cuBLAS GEMMs around one fused mixer kernel.
    """

    def __init__(self, cfg: HyenaConfig, dtype: torch.dtype = torch.bfloat16, dev=None):
        self.cfg = cfg
        self.dtype = dtype
        self.dev = dev or device()
        D = cfg.width
        w = [projection_dense(getattr(cfg, n)) for n in ("w_q", "w_k", "w_v")]
        self.w_qkv_t = torch.from_numpy(np.concatenate([m.T for m in w], axis=0)).to(self.dev, dtype).contiguous()
        self.w_out_t = torch.from_numpy(np.ascontiguousarray(projection_dense(cfg.w_out).T)).to(self.dev, dtype)
        # fp32 projections on the tensor cores (blas.py: three-way bf16 split, six bf16 GEMMs);
        # HY_FP32_GEMM=simt keeps cuBLAS's CUDA-core fp32 GEMM
        self.split3 = dtype == torch.float32 and os.environ.get("HY_FP32_GEMM", "split3") == "split3"
        if self.split3:
            self.w_qkv_parts = blas.split3_weight(self.w_qkv_t)
            self.w_out_parts = blas.split3_weight(self.w_out_t.contiguous())
        tdt = ops.tap_dtype(dtype)
        self.lhf = max(cfg.q_feat.filter_len, cfg.k_feat.filter_len, cfg.v_feat.filter_len)
        feat = np.zeros((3, D, self.lhf))
        for i, bank in enumerate((cfg.q_feat, cfg.k_feat, cfg.v_feat)):
            feat[i, :, :bank.filter_len] = bank.taps_per_channel()
        self.feat_taps = torch.from_numpy(feat).to(self.dev, tdt).contiguous()
        self.feat_packed = ops.feat_pack(self.feat_taps) if dtype == torch.bfloat16 else None
        inner = cfg.inner
        self.gs = inner.group_size
        self.lh = inner.filter_len
        self.decay = None
        self.li_modes = None
        self.li_scan_modes = None
        if isinstance(inner.filters[0], ImplicitFilter):
            self.inner_taps = None  # materialised lazily (short-filter fused path only)
            npoles = {f.poles.size for f in inner.filters}
            npmax = max(npoles)
            if npmax <= LI_SCAN_MAX_POLES:
                # (residues, poles) fp64 for the modal scan (hy_li_scan_fwd): the reference-
                # precision LI path; ragged pole counts padded with R = 0, lam = 0 modes
                res = np.zeros((inner.n_groups, npmax))
                pol = np.zeros((inner.n_groups, npmax))
                for g, f in enumerate(inner.filters):
                    res[g, :f.poles.size] = f.residues
                    pol[g, :f.poles.size] = f.poles
                self.li_scan_modes = (torch.from_numpy(res).to(self.dev), torch.from_numpy(pol).to(self.dev))
            if dtype == torch.bfloat16 and len(npoles) == 1 and max(npoles) <= 8:
                # (residues, poles) per group for the tcgen05 implicit-filter kernel
                self.li_modes = (torch.tensor(np.stack([f.residues for f in inner.filters]), dtype=torch.float32,
                                              device=self.dev),
                                 torch.tensor(np.stack([f.poles for f in inner.filters]), dtype=torch.float32,
                                              device=self.dev))
        elif isinstance(inner.filters[0], RegularizedFilter) and dtype != torch.float64:
            # taps_hat + per-group rate*log2(base): the decay is applied inside the kernels
            self.inner_taps = torch.from_numpy(np.stack([f.taps_hat for f in inner.filters])).to(self.dev, tdt)
            self.decay = torch.tensor([f.decay_rate * np.log2(f.base) for f in inner.filters],
                                      dtype=torch.float32, device=self.dev)
        else:
            self.inner_taps = torch.from_numpy(inner.materialized()).to(self.dev, tdt)
        self._mat_taps = None
        # the projection GEMM with the featurizers and u = fk * fv in its
        # epilogue (hy_qkv_feat_gemm), then the gated inner conv reads (fq, u); HY_QKV_FUSED=1
        # selects it (cuBLAS + the fused mixer stays the default: DESIGN §3.6)
        self.qkv_fused = os.environ.get("HY_QKV_FUSED", "0") == "1"
        self._w_perm = None

    def qkv_fused_eligible(self, L: int) -> bool:
        if self.dtype != torch.bfloat16 or self.cfg.width % 128 or L % 256 or self.lhf > 8:
            return False
        return self.li_modes is not None or (self.inner_taps is not None and self.lh <= ops.BLOCK_CONV_MAX_LH)

    def project_featurized(self, x3: torch.Tensor):
        """(fq, u), each (B, D, L): hyena.py:122-126 and the gate product k * v of :184 in one
        tcgen05 GEMM whose epilogue runs the featurizer FIRs (bf16)."""
        if self._w_perm is None:
            self._w_perm = ops.qkv_weight_permute(self.w_qkv_t)
        return ops.qkv_feat_gemm(x3, self._w_perm, self.feat_taps)

    def inner_gated(self, u: torch.Tensor, fq: torch.Tensor) -> torch.Tensor:
        """fq * inner(u) (hyena.py:183-186) on the fused projections."""
        if self.li_modes is not None:
            return ops.li_conv(u, self.li_modes[0], self.li_modes[1], self.gs, q=fq)
        if self.lh <= 129:  # T0 / T1 on the 32-chunk kernel (0.167 ms at C2 vs 0.183 on the K-block one)
            return ops.two_stage(u, self.inner_taps, self.gs, q=fq, decay=self.decay)
        return ops.block_conv(u, self.inner_taps, self.gs, q=fq, decay=self.decay)

    @property
    def materialized_inner(self) -> torch.Tensor:
        if self.inner_taps is None:
            self.inner_taps = _implicit_taps_device(self.cfg.inner, self.dev, ops.tap_dtype(self.dtype))
        if self.decay is None:
            return self.inner_taps
        if self._mat_taps is None:
            t = torch.arange(self.lh, device=self.dev, dtype=torch.float32)
            self._mat_taps = (self.inner_taps * torch.exp2(-self.decay[:, None] * t[None, :])).contiguous()
        return self._mat_taps

    def mixer(self, proj: torch.Tensor) -> torch.Tensor:
        """q * inner(k * v) from the (B, 3D, L) projections."""
        D = self.cfg.width
        if self.li_modes is not None and proj.shape[-1] % 8 == 0:
            return ops.li_mixer(proj, self.feat_taps, self.li_modes[0], self.li_modes[1], self.gs,
                                packed=self.feat_packed)
        if self.li_scan_modes is not None and self.lhf <= 8:
            # LI at the reference's precision (fp32 / fp64), > 8 poles or L % 8 != 0: featurizers,
            # gates and exact per-mode state scans in one pass (no FFT, no length-L filter)
            return ops.li_scan_mixer(proj, self.feat_taps, self.li_scan_modes[0], self.li_scan_modes[1], self.gs)
        if fused_mixer_eligible(self.dtype, self.lh, proj.shape[-1]):
            # LI keeps no explicit taps (modal form); a short LI filter is materialised once
            taps = self.inner_taps if self.inner_taps is not None else self.materialized_inner
            return ops.hyena_mixer(proj, self.feat_taps, taps, self.gs, decay=self.decay,
                                   packed=self.feat_packed)
        B, _, L = proj.shape
        if self.dtype == torch.bfloat16 and 129 < self.lh <= ops.BLOCK_CONV_MAX_LH and L % 8 == 0 \
                and self.inner_taps is not None and self.lhf <= 8:
            # long explicit / MR filters: one featurizer stream (u = fk * fv, fq), then the K-block
            # tcgen05 conv gated by fq (K + 1 spill factors, blockconv.py:103-121)
            u, fq = ops.featurize(proj, self.feat_taps)
            return ops.block_conv(u, self.inner_taps, self.gs, q=fq, decay=self.decay)
        # unfused: featurizers over all 3D rows in one launch, then the gated inner conv
        feats = ops.causal_conv(proj, self.feat_taps.reshape(3 * D, self.lhf), 1)
        q, k, v = (feats[:, i * D:(i + 1) * D].contiguous() for i in range(3))
        if self.li_scan_modes is not None:  # featurizers longer than 8 taps: exact modal scans
            return ops.li_scan(v, self.li_scan_modes[0], self.li_scan_modes[1], self.gs, q=q, k=k)
        if self.lh > 129 or self.cfg.variant == "LI":
            if self.dtype != torch.float64 and getattr(self, "_spec_L", None) != L:
                # the filter half of the FFT conv is a parameter transform: once per length
                self._spec = ops.fft_spectrum(self.materialized_inner, L)
                self._spec_L = L
            return ops.long_conv(v, self.materialized_inner, self.gs, q=q, k=k,
                                 spectrum=self._spec if self.dtype != torch.float64 else None)
        return ops.gated_conv(v, self.materialized_inner, self.gs, q=q, k=k)

    def forward(self, x: torch.Tensor, events=None, accumulate_into: torch.Tensor | None = None) -> torch.Tensor:
        """events: optional (start, end) CUDA events recorded around the mixer kernel.
        accumulate_into: a caller-owned tensor of the output's shape (e.g. x itself in a residual
        stack); the result is added into it in the out-projection GEMM's epilogue (beta = 1) and
        it is returned — the residual add costs no separate pass."""
        squeeze = x.dim() == 2
        x3 = x.unsqueeze(0) if squeeze else x
        if x3.shape[1] != self.cfg.width:
            raise ValueError(f"input has {x3.shape[1]} channels, operator width is {self.cfg.width}")
        if self.cfg.variant == "LI" and self.lh != x3.shape[2]:
            raise ValueError(
                f"LI inner filter length {self.lh} must equal the sequence length {x3.shape[2]}")
        if x3.dtype != self.dtype:
            raise ValueError(f"operator packed for {self.dtype}, got {x3.dtype}")
        if self.qkv_fused and self.qkv_fused_eligible(x3.shape[2]):
            fq, u = self.project_featurized(x3)
            if events is not None:
                events[0].record()
            mixed = self.inner_gated(u, fq)
        else:
            proj = self.project(x3)
            if events is not None:
                events[0].record()
            mixed = self.mixer(proj)
        if events is not None:
            events[1].record()
        acc = None
        if accumulate_into is not None:
            if tuple(accumulate_into.shape) != tuple(x.shape) or accumulate_into.dtype != self.dtype:
                raise ValueError("accumulate_into must match the output's shape and dtype")
            acc = accumulate_into.unsqueeze(0) if squeeze else accumulate_into
        y = self.out_project(mixed, acc)
        return y[0] if squeeze else y

    def project(self, x3: torch.Tensor) -> torch.Tensor:
        """(B, 3D, L) = W_qkv^T x (hyena.py:122-124)."""
        if self.split3:
            return blas.matmul_split3(self.w_qkv_parts, blas.split3_act(x3))
        return torch.matmul(self.w_qkv_t, x3)

    def out_project(self, mixed: torch.Tensor, acc: torch.Tensor | None = None) -> torch.Tensor:
        """y = W_out^T mixed (hyena.py:188); with acc: acc += W_out^T mixed in the GEMM epilogue
        (the residual of hyena.py:405), returned."""
        if self.split3:
            return blas.matmul_split3(self.w_out_parts, blas.split3_act(mixed), out=acc, accumulate=acc is not None)
        if acc is None:
            return torch.matmul(self.w_out_t, mixed)
        if acc.shape[0] == 1:
            acc[0].addmm_(self.w_out_t, mixed[0])
        else:
            acc.baddbmm_(self.w_out_t.expand(acc.shape[0], -1, -1), mixed)
        return acc

    __call__ = forward


_OPS: dict = {}


def operator_for(cfg: HyenaConfig, dtype: torch.dtype) -> HyenaOperator:
    """Cached device packing of a config (evicted when the config is garbage collected)."""
    key = (id(cfg), dtype)
    hit = _OPS.get(key)
    if hit is not None and hit[0]() is cfg:
        return hit[1]
    op = HyenaOperator(cfg, dtype)
    _OPS[key] = (weakref.ref(cfg, lambda _r, k=key: _OPS.pop(k, None)), op)
    return op


def _fp32_exact():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False


def hyena_forward(x: SeqTensor, cfg: HyenaConfig) -> SeqTensor:
    """Eq. 1, y = W_out^T (q * conv_inner(k * v)) (hyena.py:157-190), on the GPU."""
    _check_input(x, cfg)
    _fp32_exact()
    xd = to_device(x)
    y = operator_for(cfg, xd.dtype).forward(xd)
    return from_device(y, x.dtype)


def _check_input(x: SeqTensor, cfg: HyenaConfig) -> None:
    if x.channels != cfg.width:
        raise ValueError(f"input has {x.channels} channels, operator width is {cfg.width}")
    if cfg.variant == "LI" and cfg.inner.filter_len != x.length:
        raise ValueError(
            f"LI inner filter length {cfg.inner.filter_len} must equal the sequence length {x.length}")


@dataclass
class HyenaSaved:
    """Forward intermediates (hyena.py:138-154), host copies."""

    cfg: HyenaConfig
    x: np.ndarray
    proj_q: np.ndarray
    proj_k: np.ndarray
    proj_v: np.ndarray
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    gated: np.ndarray
    conv_out: np.ndarray
    mixed: np.ndarray
    ts_saved: object
    dtype: str


def hyena_forward_saved(x: SeqTensor, cfg: HyenaConfig):
    """Forward half of hyena.py:162-190 returning (y, HyenaSaved) with the intermediates."""
    _check_input(x, cfg)
    _fp32_exact()
    xd = to_device(x)
    op = operator_for(cfg, xd.dtype)
    D = cfg.width
    proj = op.project(xd.unsqueeze(0))[0] if op.split3 else torch.matmul(op.w_qkv_t, xd)
    feats = ops.causal_conv(proj, op.feat_taps.reshape(3 * D, op.lhf), 1)
    q, k, v = (feats[i * D:(i + 1) * D].contiguous() for i in range(3))
    gated = k * v
    if op.li_scan_modes is not None:
        conv_out = ops.li_scan(gated, op.li_scan_modes[0], op.li_scan_modes[1], op.gs)
    elif op.lh > 129:
        conv_out = ops.long_conv(gated, op.materialized_inner, op.gs)
    else:
        conv_out = ops.gated_conv(gated, op.materialized_inner, op.gs)
    mixed = q * conv_out
    y = op.out_project(mixed.unsqueeze(0))[0] if op.split3 else torch.matmul(op.w_out_t, mixed)
    h = lambda t: t.detach().cpu().numpy().astype(np.float64)  # noqa: E731
    saved = HyenaSaved(cfg, h(xd), h(proj[:D]), h(proj[D:2 * D]), h(proj[2 * D:]), h(q), h(k), h(v), h(gated),
                       h(conv_out), h(mixed), None, x.dtype)
    return from_device(y, x.dtype), saved


# ---------------------------------------------------------------- layouts (hyena.py:350-417)


@dataclass(frozen=True, eq=False)
class LayoutSpec:
    """Variant pattern repeated `depth` times with one config per layer."""

    pattern: tuple
    depth: int
    layers: tuple

    def __post_init__(self):
        pattern = tuple(self.pattern)
        layers = tuple(self.layers)
        if not pattern:
            raise ValueError("pattern must be nonempty")
        for v in pattern:
            if v not in VARIANTS:
                raise ValueError(f"unknown variant {v!r} in pattern")
        if self.depth < 1:
            raise ValueError("depth must be >= 1")
        if len(layers) != len(pattern) * self.depth:
            raise ValueError(f"need {len(pattern) * self.depth} layer configs "
                             f"(pattern {len(pattern)} x depth {self.depth}), got {len(layers)}")
        for i, cfg in enumerate(layers):
            want = pattern[i % len(pattern)]
            if cfg.variant != want:
                raise ValueError(f"layer {i} has variant {cfg.variant}, pattern expects {want}")
        object.__setattr__(self, "pattern", pattern)
        object.__setattr__(self, "layers", layers)


@dataclass(frozen=True, eq=False)
class OperatorStack:
    layers: tuple
    residual: bool = False


def build_layout(spec: LayoutSpec, residual: bool = False) -> OperatorStack:
    widths = {cfg.width for cfg in spec.layers}
    if len(widths) != 1:
        raise ValueError(f"layer widths differ: {sorted(widths)}")
    return OperatorStack(tuple(spec.layers), residual=residual)


def layout_forward_device(x: torch.Tensor, stack: OperatorStack) -> torch.Tensor:
    """Torch-native stack forward: activations stay on the device between layers. The residual
    add (hyena.py:405) is fused into each layer's out-projection GEMM (beta = 1) on a buffer the
    stack owns; the caller's x is never written."""
    cur = x
    for i, cfg in enumerate(stack.layers):
        op = operator_for(cfg, x.dtype)
        if stack.residual:
            cur = op.forward(cur, accumulate_into=cur.clone() if i == 0 else cur)
        else:
            cur = op.forward(cur)
    return cur


def layout_forward(x: SeqTensor, stack: OperatorStack) -> SeqTensor:
    """Sequential composition with optional residual (hyena.py:394-406)."""
    for cfg in stack.layers:
        _check_input(x, cfg)
    _fp32_exact()
    return from_device(layout_forward_device(to_device(x), stack), x.dtype)


def layout_forward_saved(x: SeqTensor, stack: OperatorStack):
    saveds = []
    cur = x
    for cfg in stack.layers:
        out, saved = hyena_forward_saved(cur, cfg)
        saveds.append(saved)
        cur = SeqTensor(cur.data + out.data, dtype=x.dtype) if stack.residual else out
    return cur, saveds


# ---------------------------------------------------------------- seeded builders (hyena.py:423-533)

DEFAULT_FEATURIZER_LEN = 7
DEFAULT_SE_LEN = 7
DEFAULT_MR_LEN = 128
DEFAULT_LI_POLES = 8
DECAY_SWEEP = (0.01, 2.0)


def _rand_taps(rng: np.random.Generator, lh: int) -> np.ndarray:
    return rng.standard_normal(lh) / np.sqrt(lh)


def _explicit_bank(rng, width: int, group_size: int, lh: int) -> GroupSpec:
    n = width // group_size
    return GroupSpec(width, group_size, tuple(ExplicitFilter(_rand_taps(rng, lh)) for _ in range(n)))


def make_inner_bank(variant: str, width: int, group_size: int, rng: np.random.Generator,
                    filter_len: int | None = None, seq_len: int | None = None,
                    n_poles: int = DEFAULT_LI_POLES, decay_base: float = 2.0) -> GroupSpec:
    """Inner bank with the reference's draw order and MR decay sweep (hyena.py:439-469)."""
    n = width // group_size
    if variant == "SE":
        return _explicit_bank(rng, width, group_size, DEFAULT_SE_LEN if filter_len is None else filter_len)
    if variant == "MR":
        lh = DEFAULT_MR_LEN if filter_len is None else filter_len
        rates = np.linspace(DECAY_SWEEP[0], DECAY_SWEEP[1], n)
        return GroupSpec(width, group_size, tuple(
            RegularizedFilter(_rand_taps(rng, lh), float(rates[g]), decay_base) for g in range(n)))
    if variant == "LI":
        if seq_len is None:
            raise ValueError("LI inner filters need the sequence length")
        filters = []
        for _ in range(n):
            poles = rng.uniform(-0.95, 0.95, size=n_poles)
            residues = rng.standard_normal(n_poles) / n_poles
            filters.append(ImplicitFilter(residues, poles, seq_len))
        return GroupSpec(width, group_size, tuple(filters))
    raise ValueError(f"variant must be one of {VARIANTS}, got {variant!r}")


def make_hyena_config(variant: str, width: int, rng: np.random.Generator, seq_len: int | None = None,
                      group_size: int = 1, featurizer_len: int = DEFAULT_FEATURIZER_LEN,
                      inner_len: int | None = None, block_size: int = 16, backend: str = "blocked",
                      n_poles: int = DEFAULT_LI_POLES) -> HyenaConfig:
    """Seeded config with the reference's exact draw order (hyena.py:472-497)."""
    scale = 1.0 / np.sqrt(width)
    projs = [rng.standard_normal((width, width)) * scale for _ in range(4)]
    return HyenaConfig(
        variant=variant, width=width,
        w_q=projs[0], w_k=projs[1], w_v=projs[2], w_out=projs[3],
        q_feat=_explicit_bank(rng, width, group_size, featurizer_len),
        k_feat=_explicit_bank(rng, width, group_size, featurizer_len),
        v_feat=_explicit_bank(rng, width, group_size, featurizer_len),
        inner=make_inner_bank(variant, width, group_size, rng, filter_len=inner_len, seq_len=seq_len,
                              n_poles=n_poles),
        block_size=block_size, backend=backend)


def make_layout(pattern, depth: int, width: int, rng: np.random.Generator, seq_len: int | None = None,
                **cfg_kw) -> LayoutSpec:
    """(hyena.py:500-513)."""
    pattern = tuple(pattern)
    layers = tuple(make_hyena_config(pattern[i % len(pattern)], width, rng, seq_len=seq_len, **cfg_kw)
                   for i in range(len(pattern) * depth))
    return LayoutSpec(pattern, depth, layers)


def identity_config(variant: str = "SE", width: int = 1, inner: GroupSpec | None = None,
                    backend: str = "direct", block_size: int = 16) -> HyenaConfig:
    """Identity projections and unit featurizers (hyena.py:516-533)."""
    eye = np.eye(width)
    unit = GroupSpec(width, width, (ExplicitFilter(np.array([1.0])),))
    return HyenaConfig(variant=variant, width=width, w_q=eye, w_k=eye.copy(), w_v=eye.copy(),
                       w_out=eye.copy(), q_feat=unit, k_feat=unit, v_feat=unit,
                       inner=unit if inner is None else inner, block_size=block_size, backend=backend)


def update_param(cfg: HyenaConfig, path: tuple, value: np.ndarray) -> HyenaConfig:
    """Functional single-leaf update (hyena.py:331-344); returns a new config."""
    from dataclasses import replace
    if path[0].startswith("w_"):
        proj = getattr(cfg, path[0])
        if len(path) == 2:
            proj = (value, proj[1]) if path[1] == "left" else (proj[0], value)
        else:
            proj = value
        return replace(cfg, **{path[0]: proj})
    role, idx, leaf = path
    groups: GroupSpec = getattr(cfg, role)
    filters = list(groups.filters)
    f = filters[idx]
    if isinstance(f, ExplicitFilter):
        filters[idx] = ExplicitFilter(value)
    elif isinstance(f, RegularizedFilter):
        filters[idx] = RegularizedFilter(value, f.decay_rate, f.base)
    elif leaf == "residues":
        filters[idx] = ImplicitFilter(value, f.poles, f.length)
    else:
        filters[idx] = ImplicitFilter(f.residues, value, f.length)
    return replace(cfg, **{role: GroupSpec(groups.channels, groups.group_size, tuple(filters))})


__all__ = [
    "VARIANTS", "BACKENDS", "MAX_SHORT_FILTER", "HyenaConfig", "HyenaOperator", "HyenaSaved",
    "LayoutSpec", "OperatorStack", "build_layout", "hyena_forward", "hyena_forward_saved",
    "identity_config", "layout_forward", "layout_forward_device", "layout_forward_saved",
    "make_hyena_config", "make_inner_bank", "make_layout", "operator_for", "projection_dense",
    "spill_count", "update_param",
]
