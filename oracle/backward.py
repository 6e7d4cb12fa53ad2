"""numpy restatement of the reference BACKWARD pass (TEST INFRASTRUCTURE ONLY).

Paths relative to /root/reference/pkg/src/convhybrid/. Like the reference, every gradient
is float64 arithmetic on the float64 intermediates the forward kept (hyena.py:138-154,
blockconv.py:139-149); the f32 forward rounds exactly where the reference's does.
Parameter-gradient containers mirror the reference: projections are arrays or
(left, right) tuples, filter grads are per role a list over groups of {leaf: array}.
"""

from __future__ import annotations

import numpy as np

from .ref import (
    F32,
    F64,
    _chunk,
    _round,
    _two_factor,
    _unchunk,
    bank_filter_len,
    bank_taps_per_channel,
    block_conv,
    direct_causal_conv,
    fft_conv,
    materialize,
    projection_dense,
    spill_count,
    two_stage_core,
)

# --------------------------------------------------------------------------
# conv adjoints (core.py:245-268)


def causal_conv_input_grad(dy: np.ndarray, taps_per_channel: np.ndarray) -> np.ndarray:
    """dx[t] = sum_j h[j] dy[t+j] (core.py:245-252)."""
    dy = np.asarray(dy, dtype=F64)
    d, length = dy.shape
    out = np.empty_like(dy)
    for ch in range(d):
        rev = np.convolve(dy[ch][::-1], np.asarray(taps_per_channel[ch], dtype=F64))[:length]
        out[ch] = rev[::-1]
    return out


def causal_conv_taps_grad(dy: np.ndarray, x: np.ndarray, bank: dict) -> np.ndarray:
    """dh[g, j] = sum_{ch in g} sum_t dy[ch, t] x[ch, t-j]; lags >= L stay 0 (core.py:255-268)."""
    dy = np.asarray(dy, dtype=F64)
    x = np.asarray(x, dtype=F64)
    d, length = dy.shape
    lh = bank_filter_len(bank)
    gs = bank["group_size"]
    out = np.zeros((len(bank["filters"]), lh))
    for ch in range(d):
        corr = np.convolve(dy[ch], x[ch][::-1])
        seg = corr[length - 1: length - 1 + lh]
        out[ch // gs, : seg.size] += seg
    return out


# --------------------------------------------------------------------------
# two-stage (blockconv.py:199-264)


def two_stage_forward_saved(v, bank: dict, lb: int, q=None, k=None):
    """(y, saved) with saved = dict(v, q, k, bank, lb, u, c) (blockconv.py:199-220)."""
    v = np.asarray(v)
    dtype = F32 if v.dtype == F32 else F64
    u = np.asarray(v, dtype=F64)
    if k is not None:
        u = u * np.asarray(k, dtype=F64)
    c = two_stage_core(u, bank, lb)
    y = c * np.asarray(q, dtype=F64) if q is not None else c
    saved = {"v": np.asarray(v, dtype=F64), "q": None if q is None else np.asarray(q, dtype=F64),
             "k": None if k is None else np.asarray(k, dtype=F64), "bank": bank, "lb": lb, "u": u, "c": c}
    return _round(y, dtype), saved


def two_stage_backward(saved: dict, dy) -> dict:
    """Gated two-stage adjoint: transposed factors for du, two-pass filter gradient
    (per-chunk partials, reduce over chunks, scatter along the block diagonals)
    (blockconv.py:223-264). Returns dict(dv, dq, dk, dtaps)."""
    dy = np.asarray(dy, dtype=F64)
    if dy.shape != saved["u"].shape:
        raise ValueError(f"dy shape {dy.shape} does not match forward shape {saved['u'].shape}")
    bank, lb = saved["bank"], saved["lb"]
    lh = bank_filter_len(bank)
    gs = bank["group_size"]
    q, k, v = saved["q"], saved["k"], saved["v"]
    dq = dy * saved["c"] if q is not None else None
    dc = dy * q if q is not None else dy
    du = np.empty_like(saved["u"])
    dtaps = np.zeros((len(bank["filters"]), lh))
    i = np.arange(lb)[:, None]
    j = np.arange(lb)[None, :]
    for g, spec in enumerate(bank["filters"]):
        sl = slice(g * gs, (g + 1) * gs)
        b0, b1 = _two_factor(materialize(spec), lb)
        dcc = _chunk(dc[sl], lb)
        dnext = np.concatenate([dcc[1:], np.zeros_like(dcc[:1])])
        du[sl] = _unchunk(b0.T @ dcc + b1.T @ dnext, dy.shape[1])
        uc = _chunk(saved["u"][sl], lb)
        uprev = np.concatenate([np.zeros_like(uc[:1]), uc[:-1]])
        p0 = np.matmul(dcc, uc.transpose(0, 2, 1)).sum(axis=0)
        p1 = np.matmul(dcc, uprev.transpose(0, 2, 1)).sum(axis=0)
        for blk, red in ((0, p0), (1, p1)):
            lag = blk * lb + i - j
            ok = (lag >= 0) & (lag < lh)
            np.add.at(dtaps[g], lag[ok], red[ok])
    dk = du * v if k is not None else None
    dv = du * k if k is not None else du
    return {"dv": dv, "dq": dq, "dk": dk, "dtaps": dtaps}


# --------------------------------------------------------------------------
# operator (hyena.py:162-284)


def filter_param_grads(spec, dtaps: np.ndarray) -> dict:
    """Tap-space gradient pulled back to the filter's own leaves (hyena.py:193-211)."""
    kind = spec[0]
    dtaps = np.asarray(dtaps, dtype=F64)
    if kind == "explicit":
        return {"taps": dtaps.copy()}
    if kind == "regularized":
        t = np.arange(dtaps.size, dtype=F64)
        return {"taps_hat": dtaps * float(spec[3]) ** (-float(spec[2]) * t)}
    if kind == "implicit":
        residues = np.asarray(spec[1], dtype=F64)
        poles = np.asarray(spec[2], dtype=F64)
        length = int(spec[3])
        t = np.arange(length, dtype=F64)
        powers = poles[None, :] ** t[:, None]
        d_res = powers.T @ dtaps
        tp = np.zeros_like(powers)
        if length > 1:
            tp[1:] = t[1:, None] * powers[:-1]
        return {"residues": d_res, "poles": (dtaps @ tp) * residues}
    raise TypeError(f"not a filter spec: {kind!r}")


def _featurize_saved(xd, proj, bank, dtype):
    """(projected a, featurized) (hyena.py:122-126)."""
    a = projection_dense(proj).T @ xd
    b = direct_causal_conv(_round(a, dtype), bank)
    return a, np.asarray(b, dtype=F64)


def hyena_forward_saved(x, cfg: dict):
    """(y, saved) restating hyena.py:162-190; saved mirrors HyenaSaved (hyena.py:138-154)."""
    x = np.asarray(x)
    dtype = F32 if x.dtype == F32 else F64
    xd = np.asarray(x, dtype=F64)
    pq, q = _featurize_saved(xd, cfg["w_q"], cfg["q_feat"], dtype)
    pk, k = _featurize_saved(xd, cfg["w_k"], cfg["k_feat"], dtype)
    pv, v = _featurize_saved(xd, cfg["w_v"], cfg["v_feat"], dtype)
    lh = bank_filter_len(cfg["inner"])
    ts = None
    if cfg["backend"] == "blocked" and spill_count(lh, cfg["block_size"]) <= 1:
        # two_stage_forward_saved(SeqTensor(v, dtype), ..., q=SeqTensor(q), k=SeqTensor(k))
        vr, qr, kr = (np.asarray(_round(a, dtype), dtype=F64) for a in (v, q, k))
        mixed_r, ts = two_stage_forward_saved(_round(v, dtype), cfg["inner"], cfg["block_size"], q=qr, k=kr)
        ts["v"], ts["q"], ts["k"] = vr, qr, kr
        gated, conv_out = ts["u"], ts["c"]
        mixed = np.asarray(mixed_r, dtype=F64)
    else:
        gated = k * v
        if cfg["backend"] == "direct":
            conv_out = np.asarray(direct_causal_conv(_round(gated, dtype), cfg["inner"]), dtype=F64)
        elif cfg["backend"] == "blocked":
            conv_out = np.asarray(block_conv(_round(gated, dtype), cfg["inner"], cfg["block_size"]), dtype=F64)
        else:
            conv_out = fft_conv(gated, bank_taps_per_channel(cfg["inner"]))
        mixed = q * conv_out
    y = projection_dense(cfg["w_out"]).T @ mixed
    saved = {"cfg": cfg, "x": xd, "proj_q": pq, "proj_k": pk, "proj_v": pv, "q": q, "k": k, "v": v,
             "gated": gated, "conv_out": conv_out, "mixed": mixed, "ts": ts, "dtype": dtype}
    return _round(y, dtype), saved


def _projection_grad(proj, d_dense):
    """(hyena.py:227-231)."""
    if isinstance(proj, tuple):
        left, right = proj
        return (d_dense @ right.T, left.T @ d_dense)
    return d_dense


def _feat_backward(grad_out, projected, x, proj, bank):
    """(dx term, dproj, filter grads) through conv(feat, proj^T x) (hyena.py:234-247)."""
    dtaps = causal_conv_taps_grad(grad_out, projected, bank)
    da = causal_conv_input_grad(grad_out, bank_taps_per_channel(bank))
    d_dense = x @ da.T
    dx_term = projection_dense(proj) @ da
    fgrads = [filter_param_grads(bank["filters"][g], dtaps[g]) for g in range(len(bank["filters"]))]
    return dx_term, _projection_grad(proj, d_dense), fgrads


def hyena_backward(saved: dict, dy) -> dict:
    """Chain rule over the operator (hyena.py:250-284). Returns dict(dx, dw_q, dw_k, dw_v,
    dw_out, filters={role: [ {leaf: grad} per group ]})."""
    cfg = saved["cfg"]
    dy = np.asarray(dy, dtype=F64)
    if dy.shape != saved["mixed"].shape:
        raise ValueError(f"dy shape {dy.shape} does not match forward output {saved['mixed'].shape}")
    dmixed = projection_dense(cfg["w_out"]) @ dy
    dw_out = _projection_grad(cfg["w_out"], saved["mixed"] @ dy.T)
    if saved["ts"] is not None:
        tg = two_stage_backward(saved["ts"], dmixed)
        dq, dk, dv, dtaps_inner = tg["dq"], tg["dk"], tg["dv"], tg["dtaps"]
    else:
        dq = dmixed * saved["conv_out"]
        dconv = dmixed * saved["q"]
        dtaps_inner = causal_conv_taps_grad(dconv, saved["gated"], cfg["inner"])
        dgated = causal_conv_input_grad(dconv, bank_taps_per_channel(cfg["inner"]))
        dk = dgated * saved["v"]
        dv = dgated * saved["k"]
    inner = cfg["inner"]
    inner_g = [filter_param_grads(inner["filters"][g], dtaps_inner[g]) for g in range(len(inner["filters"]))]
    x = saved["x"]
    dx_q, dw_q, fq = _feat_backward(dq, saved["proj_q"], x, cfg["w_q"], cfg["q_feat"])
    dx_k, dw_k, fk = _feat_backward(dk, saved["proj_k"], x, cfg["w_k"], cfg["k_feat"])
    dx_v, dw_v, fv = _feat_backward(dv, saved["proj_v"], x, cfg["w_v"], cfg["v_feat"])
    return {"dx": dx_q + dx_k + dx_v, "dw_q": dw_q, "dw_k": dw_k, "dw_v": dw_v, "dw_out": dw_out,
            "filters": {"q_feat": fq, "k_feat": fk, "v_feat": fv, "inner": inner_g}}


def layout_forward_saved(x, layers, residual: bool = False):
    """(y, per-layer saved) (hyena.py:375-406)."""
    x = np.asarray(x)
    dtype = F32 if x.dtype == F32 else F64
    cur = x
    saveds = []
    for cfg in layers:
        out, s = hyena_forward_saved(cur, cfg)
        saveds.append(s)
        cur = _round(np.asarray(cur, dtype=F64) + np.asarray(out, dtype=F64), dtype) if residual else out
    return cur, saveds


def layout_backward(layers, saveds, dy, residual: bool = False):
    """(dx, per-layer grads), last layer first (hyena.py:409-417)."""
    dcur = np.asarray(dy, dtype=F64)
    grads = [None] * len(layers)
    for i in range(len(layers) - 1, -1, -1):
        g = hyena_backward(saveds[i], dcur)
        grads[i] = g
        dcur = dcur + g["dx"] if residual else g["dx"]
    return dcur, grads
