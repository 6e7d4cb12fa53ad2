"""Backward pass of the Hyena operator over the sm_100a kernels.

Two entry levels, like the forward:

* the reference API (hyena.py:193-284, 409-417): `hyena_backward(saved, dy)` on the host
  `HyenaSaved` context, `filter_param_grads`, `iter_params`, `grad_for_path`,
  `layout_backward`. Arithmetic is fp64 on the device (the reference differentiates in
  float64 on its float64 intermediates); conv adjoints run in hy_causal_conv_bwd.
* the torch-native device path: `operator_backward(op, x, dy)` on (B, D, L) CUDA tensors in
  the operator's dtype — cuBLAS GEMMs for the projections, hy_causal_conv_bwd for the
  featurizer and explicit / regularized inner adjoints, and for implicit (LI) filters the
  time-reversed tcgen05 modal conv for du plus the exact per-mode scans of hy_li_param_grad
  for (residues, poles) — no length-L tap gradient is ever formed.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np
import torch

from . import blas, ops
from .core import ExplicitFilter, GroupSpec, ImplicitFilter, RegularizedFilter, SeqTensor, device

# ---------------------------------------------------------------- reference API


def _f64(a) -> torch.Tensor:
    return torch.from_numpy(np.array(a, dtype=np.float64, copy=True)).to(device())


def filter_param_grads(spec, dtaps) -> dict:
    """Pull a tap-space gradient back to the filter's own leaves (hyena.py:193-211)."""
    dt = dtaps if isinstance(dtaps, torch.Tensor) else _f64(dtaps)
    dt = dt.to(torch.float64)
    if isinstance(spec, ExplicitFilter):
        return {"taps": dt.clone().cpu().numpy()}
    if isinstance(spec, RegularizedFilter):
        t = torch.arange(spec.length, dtype=torch.float64, device=dt.device)
        return {"taps_hat": (dt * torch.pow(torch.tensor(spec.base, dtype=torch.float64, device=dt.device),
                                            -spec.decay_rate * t)).cpu().numpy()}
    if isinstance(spec, ImplicitFilter):
        t = torch.arange(spec.length, dtype=torch.float64, device=dt.device)
        poles = torch.from_numpy(np.asarray(spec.poles, dtype=np.float64)).to(dt.device)
        res = torch.from_numpy(np.asarray(spec.residues, dtype=np.float64)).to(dt.device)
        powers = torch.pow(poles[None, :], t[:, None])  # (lh, n), 0**0 = 1
        d_res = powers.T @ dt
        tp = torch.zeros_like(powers)
        if spec.length > 1:
            tp[1:] = t[1:, None] * powers[:-1]
        return {"residues": d_res.cpu().numpy(), "poles": ((dt @ tp) * res).cpu().numpy()}
    raise TypeError(f"not a filter spec: {type(spec).__name__}")


@dataclass
class HyenaGrads:
    """(hyena.py:214-224)."""

    dx: np.ndarray
    dw_q: object
    dw_k: object
    dw_v: object
    dw_out: object
    filters: dict  # role -> list over groups of {param name -> gradient array}


def _projection_grad(proj, d_dense: torch.Tensor):
    """(hyena.py:227-231): dense gradient, or (left, right) for a factored projection."""
    if isinstance(proj, tuple):
        left, right = proj
        return ((d_dense @ _f64(right).T).cpu().numpy(), (_f64(left).T @ d_dense).cpu().numpy())
    return d_dense.cpu().numpy()


def _feat_backward(grad_out: torch.Tensor, projected: np.ndarray, x: torch.Tensor, proj, groups: GroupSpec):
    """(dx term, dproj, filter grads) through conv(feat, proj^T x) (hyena.py:234-247)."""
    from .hyena import projection_dense
    da, dtaps = ops.causal_conv_bwd(grad_out, _f64(projected), _f64(groups.materialized()), groups.group_size)
    d_dense = x @ da.T
    dx_term = _f64(projection_dense(proj)) @ da
    fgrads = [filter_param_grads(groups.filters[g], dtaps[g]) for g in range(groups.n_groups)]
    return dx_term, _projection_grad(proj, d_dense), fgrads


def hyena_backward(saved, dy) -> HyenaGrads:
    """Chain rule over the whole operator, all filter kinds (hyena.py:250-284), on the GPU (fp64)."""
    from .hyena import HyenaSaved, projection_dense
    if not isinstance(saved, HyenaSaved):
        raise ValueError("backward needs the HyenaSaved context from hyena_forward_saved")
    cfg = saved.cfg
    dy = dy.data if isinstance(dy, SeqTensor) else np.asarray(dy, dtype=np.float64)
    if dy.shape != saved.mixed.shape:
        raise ValueError(f"dy shape {dy.shape} does not match forward output {saved.mixed.shape}")
    dyd = _f64(dy)
    dmixed = _f64(projection_dense(cfg.w_out)) @ dyd
    dw_out = _projection_grad(cfg.w_out, _f64(saved.mixed) @ dyd.T)
    inner = cfg.inner
    dq = dmixed * _f64(saved.conv_out)
    dconv = dmixed * _f64(saved.q)
    if inner.filter_len > 2048:
        raise NotImplementedError(
            f"reference-API backward: inner filter length {inner.filter_len} > 2048 (use the device path, "
            "operator_backward, which differentiates implicit filters by per-mode scans)")
    dgated, dtaps_inner = ops.causal_conv_bwd(dconv, _f64(saved.gated), _f64(inner.materialized()),
                                              inner.group_size)
    dk = dgated * _f64(saved.v)
    dv = dgated * _f64(saved.k)
    inner_g = [filter_param_grads(inner.filters[g], dtaps_inner[g]) for g in range(inner.n_groups)]
    x = _f64(saved.x)
    dx_q, dw_q, fq = _feat_backward(dq, saved.proj_q, x, cfg.w_q, cfg.q_feat)
    dx_k, dw_k, fk = _feat_backward(dk, saved.proj_k, x, cfg.w_k, cfg.k_feat)
    dx_v, dw_v, fv = _feat_backward(dv, saved.proj_v, x, cfg.w_v, cfg.v_feat)
    return HyenaGrads(dx=(dx_q + dx_k + dx_v).cpu().numpy(), dw_q=dw_q, dw_k=dw_k, dw_v=dw_v, dw_out=dw_out,
                      filters={"q_feat": fq, "k_feat": fk, "v_feat": fv, "inner": inner_g})


def iter_params(cfg) -> Iterator[tuple[tuple, np.ndarray]]:
    """Yield (path, array) for every learnable parameter leaf of a config (hyena.py:291-309)."""
    for name in ("w_q", "w_k", "w_v", "w_out"):
        proj = getattr(cfg, name)
        if isinstance(proj, tuple):
            yield (name, "left"), proj[0]
            yield (name, "right"), proj[1]
        else:
            yield (name,), proj
    for role in ("q_feat", "k_feat", "v_feat", "inner"):
        groups: GroupSpec = getattr(cfg, role)
        for g, f in enumerate(groups.filters):
            if isinstance(f, ExplicitFilter):
                yield (role, g, "taps"), f.taps
            elif isinstance(f, RegularizedFilter):
                yield (role, g, "taps_hat"), f.taps_hat
            elif isinstance(f, ImplicitFilter):
                yield (role, g, "residues"), f.residues
                yield (role, g, "poles"), f.poles


def grad_for_path(grads: HyenaGrads, path: tuple) -> np.ndarray:
    """(hyena.py:312-319)."""
    if path[0].startswith("w_"):
        g = getattr(grads, "d" + path[0])
        if len(path) == 2:
            return g[0] if path[1] == "left" else g[1]
        return g
    role, idx, leaf = path
    return grads.filters[role][idx][leaf]


def layout_backward(stack, saveds: list, dy) -> tuple[np.ndarray, list]:
    """Gradient through the whole stack, last layer first; returns (dx, per-layer HyenaGrads)
    (hyena.py:409-417)."""
    dcur = dy.data if isinstance(dy, SeqTensor) else np.asarray(dy, dtype=np.float64)
    layer_grads: list = [None] * len(stack.layers)
    for i in range(len(stack.layers) - 1, -1, -1):
        g = hyena_backward(saveds[i], dcur)
        layer_grads[i] = g
        dcur = (_f64(dcur) + _f64(g.dx)).cpu().numpy() if stack.residual else g.dx
    return dcur, layer_grads


# ---------------------------------------------------------------- device path


@dataclass
class DeviceGrads:
    """Gradients of sum(dy * op.forward(x)) w.r.t. the operator's packed device parameters.

    w_qkv_t: (3D, D) like op.w_qkv_t; w_out_t: (D, D) like op.w_out_t; feat_taps: (3, D, lhf)
    fp32; inner: {"taps": (G, lh)} for explicit, {"taps_hat": (G, lh)} for regularized,
    {"residues", "poles": (G, n)} for implicit filters (fp32; fp64 for fp64 operators)."""

    w_qkv_t: torch.Tensor
    w_out_t: torch.Tensor
    feat_taps: torch.Tensor
    inner: dict


def _batched_outer(a: torch.Tensor, b: torch.Tensor, split3: bool = False) -> torch.Tensor:
    """sum_b a[b] @ b[b]^T for (B, M, L) x (B, N, L): cuBLAS GEMMs accumulating in an fp32 output
    (fp64 for fp64 inputs) across the batch (beta = 1), no separate conversion / add passes."""
    if a.dtype == torch.float64:
        out = torch.matmul(a[0], b[0].transpose(0, 1))
        for i in range(1, a.shape[0]):
            out.addmm_(a[i], b[i].transpose(0, 1))
        return out
    if a.dtype == torch.float32 and split3:
        # fp32 on the bf16 tensor cores (blas.py: exact three-way splits, fp32 accumulation)
        out = None
        for i in range(a.shape[0]):
            out = blas.matmul_split3(blas.split3(a[i]), blas.split3(b[i].transpose(0, 1)), out=out,
                                     accumulate=i > 0)
        return out
    kw = {} if a.dtype == torch.float32 else {"out_dtype": torch.float32}
    out = torch.mm(a[0], b[0].transpose(0, 1), **kw)
    for i in range(1, a.shape[0]):
        torch.addmm(out, a[i], b[i].transpose(0, 1), out=out, **kw)
    return out


def operator_backward(op, x: torch.Tensor, dy: torch.Tensor, proj: torch.Tensor | None = None, events=None):
    """(dx, DeviceGrads) for y = op.forward(x) and upstream gradient dy, both (B, D, L) CUDA
    tensors of the operator's dtype. Recomputes the mixer intermediates from the projections
    (pass `proj` = op.w_qkv_t @ x to skip that GEMM). Same chain rule as hyena.py:250-284.
    events: optional {"inner_taps": (start, end), "featurizer_bwd": (start, end)} CUDA events
    recorded around those kernels (bench accounting)."""

    def mark(name, i):
        if events is not None and name in events:
            events[name][i].record()
    squeeze = x.dim() == 2
    x3 = x.unsqueeze(0) if squeeze else x
    dy3 = dy.unsqueeze(0) if squeeze else dy
    D = op.cfg.width
    if x3.shape[1] != D or dy3.shape != x3.shape or x3.dtype != op.dtype or dy3.dtype != op.dtype:
        raise ValueError("x and dy must be (B, D, L) tensors of the operator's dtype")
    B, _, L = x3.shape
    if proj is None:
        proj = op.project(x3)
    inner = op.cfg.inner
    implicit = isinstance(inner.filters[0], ImplicitFilter)
    npoles = {f.poles.size for f in inner.filters} if implicit else set()
    scan = implicit and op.dtype != torch.float64 and len(npoles) == 1 and max(npoles) <= 8
    modal = scan and op.dtype == torch.bfloat16 and L % 8 == 0
    if scan:
        res = torch.tensor(np.stack([f.residues for f in inner.filters]), dtype=torch.float32, device=x3.device)
        poles = torch.tensor(np.stack([f.poles for f in inner.filters]), dtype=torch.float32, device=x3.device)
    ts_ok = op.dtype == torch.bfloat16 and op.lh <= 129 and L % 8 == 0 and op.inner_taps is not None \
        and not implicit
    # longer explicit / MR filters: the K-block tcgen05 conv (forward c and the reversed-time du)
    kb_ok = op.dtype == torch.bfloat16 and 129 < op.lh <= ops.BLOCK_CONV_MAX_LH and L % 8 == 0 \
        and op.inner_taps is not None and not implicit

    def inner_conv(a):
        if modal:
            return ops.li_conv(a, res, poles, op.gs)
        if ts_ok:
            return ops.two_stage(a, op.inner_taps, op.gs, decay=op.decay)
        if kb_ok:
            return ops.block_conv(a, op.inner_taps, op.gs, decay=op.decay)
        if op.cfg.variant == "LI" and op.li_scan_modes is not None:
            return ops.li_scan(a, op.li_scan_modes[0], op.li_scan_modes[1], op.gs)  # exact modal scans
        if op.lh > 129 or op.cfg.variant == "LI":
            return ops.long_conv(a, op.materialized_inner, op.gs)
        return ops.gated_conv(a, op.materialized_inner, op.gs)

    def wt_mm(name, w_t, rhs):  # W^T-side products: W (= w_t^T) @ rhs, fp32 via split-bf16
        if not op.split3:
            return torch.matmul(w_t.transpose(0, 1), rhs)
        parts = getattr(op, name, None)
        if parts is None:
            parts = blas.split3_weight(w_t.transpose(0, 1).contiguous())
            setattr(op, name, parts)
        return blas.matmul_split3(parts, blas.split3_act(rhs))

    dmixed = wt_mm("_w_out_bwd_parts", op.w_out_t, dy3)
    fused = op.dtype != torch.float64 and op.lhf <= 8 and L % 8 == 0
    rev = fused and (modal or ts_ok or kb_ok)  # du runs as the causal tcgen05 conv of the reversed dc
    dc_rev = None
    if fused:
        # featurizers recomputed in-stream: u = fk * fv and dc = dmixed * fq, one pass
        if rev:
            u, dc, dc_rev = ops.mixer_bwd_prep(proj, dmixed, op.feat_taps, reversed_dc=True)
        else:
            u, dc = ops.mixer_bwd_prep(proj, dmixed, op.feat_taps)
        c = inner_conv(u)
        mixed = op.mixer(proj) if (modal or ts_ok or kb_ok) else None  # fused tcgen05 forward mixer
        if mixed is None:
            mixed = ops.causal_conv(proj[:, :D].contiguous(), op.feat_taps[0], 1) * c
    else:
        feats = ops.causal_conv(proj, op.feat_taps.reshape(3 * D, op.lhf), 1)
        q, k, v = feats[:, :D], feats[:, D:2 * D], feats[:, 2 * D:]
        u = k * v
        c = inner_conv(u)
        mixed = q * c
        dc = dmixed * q
    g_out = _batched_outer(dy3, mixed, op.split3)
    inner_g = {}
    du_rev = None  # du stored time-reversed (consumed mirrored by the featurizer backward)
    if scan:
        # du[t] = sum_{s >= t} h[s - t] dc[s]: the causal conv of the time-reversed dc
        if rev:
            du_rev = inner_conv(dc_rev)
        else:
            rdc = torch.flip(dc, dims=[-1]).contiguous()
            rdu = ops.li_conv(rdc, res, poles, op.gs) if modal else inner_conv(rdc)
            du = torch.flip(rdu, dims=[-1])
        mark("inner_taps", 0)
        inner_g["residues"], inner_g["poles"] = ops.li_param_grad(dc, u, res, poles, op.gs)
        mark("inner_taps", 1)
    else:
        taps = op.materialized_inner
        if taps.shape[-1] > 2048:
            raise NotImplementedError(f"device backward: inner filter of {taps.shape[-1]} taps > 2048 "
                                      "(implicit filters use the per-mode scans for fp32 / bf16)")
        if ts_ok:
            # du = anti-causal conv of dc = the causal two-stage conv (tcgen05, transposed
            # factors become the forward factors) of the time-reversed dc
            rdc = dc_rev if rev else torch.flip(dc, dims=[-1]).contiguous()
            rdu = ops.two_stage(rdc, op.inner_taps, op.gs, decay=op.decay)
            if rev:
                du_rev = rdu
            else:
                du = torch.flip(rdu, dims=[-1])
            mark("inner_taps", 0)
            dtaps = ops.two_stage_taps_grad(dc, u, op.lh, op.gs)  # tcgen05, both passes fused
            mark("inner_taps", 1)
        elif kb_ok:
            # du as the causal K-block conv of the reversed dc (the transposed factors are the
            # forward factors on reversed time); the tap gradient by the generic correlation
            rdc = dc_rev if rev else torch.flip(dc, dims=[-1]).contiguous()
            rdu = ops.block_conv(rdc, op.inner_taps, op.gs, decay=op.decay)
            if rev:
                du_rev = rdu
            else:
                du = torch.flip(rdu, dims=[-1])
            _, dtaps = ops.causal_conv_bwd(dc, u, op.lh, op.gs, want_dx=False)
        else:
            du, dtaps = ops.causal_conv_bwd(dc, u, taps, op.gs)
        if implicit:  # fp64: pull the tap gradient back through h_t = sum_n R_n lam_n^t
            r64 = torch.tensor(np.stack([f.residues for f in inner.filters]), device=dtaps.device)
            p64 = torch.tensor(np.stack([f.poles for f in inner.filters]), device=dtaps.device)
            t = torch.arange(op.lh, dtype=torch.float64, device=dtaps.device)
            powers = torch.pow(p64[:, None, :], t[None, :, None])  # (G, lh, n)
            dt64 = dtaps.double()
            inner_g["residues"] = torch.einsum("gtn,gt->gn", powers, dt64).to(dtaps.dtype)
            tp = torch.zeros_like(powers)
            tp[:, 1:] = t[None, 1:, None] * powers[:, :-1]
            inner_g["poles"] = (torch.einsum("gt,gtn->gn", dt64, tp) * r64).to(dtaps.dtype)
        elif op.decay is not None:
            t = torch.arange(op.lh, device=dtaps.device, dtype=torch.float32)
            inner_g["taps_hat"] = dtaps * torch.exp2(-op.decay[:, None] * t[None, :]).to(dtaps.dtype)
        elif isinstance(inner.filters[0], RegularizedFilter):  # fp64 operators keep materialised taps
            base = torch.tensor([f.base for f in inner.filters], dtype=torch.float64, device=dtaps.device)
            rate = torch.tensor([f.decay_rate for f in inner.filters], dtype=torch.float64, device=dtaps.device)
            t = torch.arange(op.lh, dtype=torch.float64, device=dtaps.device)
            inner_g["taps_hat"] = dtaps * torch.pow(base[:, None], -rate[:, None] * t[None, :])
        else:
            inner_g["taps"] = dtaps
    if fused:
        # one pass: featurizers recomputed, gate products, anti-causal FIRs, tap gradients
        mark("featurizer_bwd", 0)
        if du_rev is not None:
            dproj, dfeat = ops.featurizer_bwd(proj, dmixed, c, du_rev, op.feat_taps, du_reversed=True)
        else:
            dproj, dfeat = ops.featurizer_bwd(proj, dmixed, c, du.contiguous(), op.feat_taps)
        mark("featurizer_bwd", 1)
    else:
        dfeats = torch.empty_like(feats)
        torch.mul(dmixed, c, out=dfeats[:, :D])                  # dq
        torch.mul(du, v, out=dfeats[:, D:2 * D])                 # dk
        torch.mul(du, k, out=dfeats[:, 2 * D:])                  # dv
        dproj, dfeat = ops.causal_conv_bwd(dfeats, proj, op.feat_taps.reshape(3 * D, op.lhf), 1)
    g_qkv = _batched_outer(dproj, x3, op.split3)
    dx = wt_mm("_w_qkv_bwd_parts", op.w_qkv_t, dproj)
    grads = DeviceGrads(w_qkv_t=g_qkv, w_out_t=g_out, feat_taps=dfeat.reshape(3, D, op.lhf), inner=inner_g)
    return (dx[0] if squeeze else dx), grads
