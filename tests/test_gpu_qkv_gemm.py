"""The projection GEMM with the featurizers in its epilogue (hy_qkv_feat_gemm, SURVEY §8(f)
rank 2) against a float64 restatement of hyena.py:122-126 + the gate product of hyena.py:184,
and the operator route that consumes it (HY_QKV_FUSED) against the oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import ops

pytestmark = pytest.mark.gpu


def _conv(x, h):
    return np.convolve(x, h)[: x.shape[-1]]


def _case(B, D, L, lhf, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((B, D, L), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((3 * D, D), device="cuda", generator=g) / np.sqrt(D)).to(torch.bfloat16)
    taps = torch.randn((3, D, lhf), device="cuda", generator=g) / 2.65
    return x, w, taps


def _want(x, w, taps, b, c):
    """fq and u of channel c, sequence b, in float64 from the same bf16 inputs."""
    D = x.shape[1]
    xb = x[b].double().cpu().numpy()
    rows = [w[i * D + c].double().cpu().numpy() @ xb for i in range(3)]
    th = taps.double().cpu().numpy()
    fq, fk, fv = (_conv(rows[i], th[i, c]) for i in range(3))
    return fq, fk * fv


@pytest.mark.parametrize("segments", [0, 1, 3, 5])
def test_qkv_feat_gemm_vs_float64(segments):
    """B = 2, D = 256, L = 1024: every tile kind (q tiles, k|v tiles), units that start
    mid-sequence (segments 3, 5: the N = 64 halo accumulation) and units that cross a sequence
    boundary; channels from every tile and both halves of the k|v tiles."""
    B, D, L = 2, 256, 1024
    x, w, taps = _case(B, D, L, 7, 1)
    out = torch.cat(ops.qkv_feat_gemm(x, ops.qkv_weight_permute(w), taps, segments=segments), dim=1)
    assert out.shape == (B, 2 * D, L)
    for b in range(B):
        for c in (0, 1, 63, 64, 100, 127, 128, 191, 200, 255):
            fq, u = _want(x, w, taps, b, c)
            assert oracle.rel_err(out[b, c].double().cpu().numpy(), fq) < 1e-2, (b, c)
            assert oracle.rel_err(out[b, D + c].double().cpu().numpy(), u) < 1e-2, (b, c)


def test_qkv_feat_gemm_segments_agree():
    """The halo accumulation (N = 64) reproduces the main tile's columns: every segmentation
    gives the same result within fp32 accumulation-order noise (bf16 outputs, 1 ulp)."""
    x, w, taps = _case(1, 384, 4096, 7, 2)
    wp = ops.qkv_weight_permute(w)
    ref = torch.cat(ops.qkv_feat_gemm(x, wp, taps, segments=1), dim=1).float()
    for s in (2, 3, 7, 16):
        got = torch.cat(ops.qkv_feat_gemm(x, wp, taps, segments=s), dim=1).float()
        assert torch.allclose(got, ref, rtol=1e-2, atol=1e-3), s


@pytest.mark.parametrize("lhf", [1, 3, 8])
def test_qkv_feat_gemm_filter_lengths(lhf):
    B, D, L = 1, 128, 512
    x, w, taps = _case(B, D, L, lhf, 3 + lhf)
    out = torch.cat(ops.qkv_feat_gemm(x, ops.qkv_weight_permute(w), taps, segments=2), dim=1)
    for c in (0, 77, 127):
        fq, u = _want(x, w, taps, 0, c)
        assert oracle.rel_err(out[0, c].double().cpu().numpy(), fq) < 1e-2
        assert oracle.rel_err(out[0, D + c].double().cpu().numpy(), u) < 1e-2


def test_qkv_feat_gemm_c2_size_properties():
    """C2 size (B = 4, D = 4096, L = 8192): scaling x by 2 scales fq by 2 and u by 4 bitwise
    (fp32 accumulation and the FIRs scale exactly), causality per 256-column tile, and sampled
    channels against float64."""
    B, D, L = 4, 4096, 8192
    x, w, taps = _case(B, D, L, 7, 4)
    wp = ops.qkv_weight_permute(w)
    y = torch.cat(ops.qkv_feat_gemm(x, wp, taps), dim=1)
    y2 = torch.cat(ops.qkv_feat_gemm(2 * x, wp, taps), dim=1)
    assert torch.equal(y2[:, :D], 2 * y[:, :D])
    assert torch.equal(y2[:, D:], 4 * y[:, D:])
    xp = x.clone()
    xp[:, :, 5000] += 1.0
    yp = torch.cat(ops.qkv_feat_gemm(xp, wp, taps), dim=1)
    assert torch.equal(yp[..., :5000], y[..., :5000])
    for b, c in ((0, 0), (1, 2047), (3, 4095), (2, 1234)):
        fq, u = _want(x, w, taps, b, c)
        assert oracle.rel_err(y[b, c].double().cpu().numpy(), fq) < 1e-2, (b, c)
        assert oracle.rel_err(y[b, D + c].double().cpu().numpy(), u) < 1e-2, (b, c)


def test_qkv_feat_gemm_rejects():
    x, w, taps = _case(1, 128, 512, 7, 5)
    with pytest.raises(ValueError):
        ops.qkv_feat_gemm(x[..., :300].contiguous(), ops.qkv_weight_permute(w), taps)
    with pytest.raises(NotImplementedError):
        ops.qkv_feat_gemm(x, ops.qkv_weight_permute(w), torch.zeros((3, 128, 9), device="cuda"))
    # the C-ABI checks TMA / vector-store alignment of its raw pointers
    from paper_2503_01868_b200 import _lib
    buf = torch.empty(2 * 128 * 512 + 8, device="cuda", dtype=torch.bfloat16)
    wp = ops.qkv_weight_permute(w)
    taps32 = taps.float().contiguous()
    st = _lib.load().hy_qkv_feat_gemm(wp.data_ptr(), x.data_ptr(), taps32.data_ptr(), 7, buf.data_ptr() + 2,
                                      buf.data_ptr() + 2 + 128 * 512 * 2, 1, 128, 512, 0, _lib.HY_BF16, 0)
    assert st == _lib.HY_ERR_INVALID


def _bf16(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def _rounded_cfg(variant, D, L, seed, **kw):
    cfg = hy.make_hyena_config(variant, D, hy.make_rng(seed), seq_len=L, **kw)
    rnd = {n: _bf16(getattr(cfg, n)) for n in ("w_q", "w_k", "w_v", "w_out")}

    def rbank(g):
        fs = []
        for f in g.filters:
            if isinstance(f, hy.ExplicitFilter):
                fs.append(hy.ExplicitFilter(_bf16(f.taps)))
            elif isinstance(f, hy.RegularizedFilter):
                fs.append(hy.RegularizedFilter(_bf16(f.taps_hat), f.decay_rate, f.base))
            else:
                fs.append(f)
        return hy.GroupSpec(g.channels, g.group_size, tuple(fs))
    return hy.HyenaConfig(**{**cfg.__dict__, **rnd, **{n: rbank(getattr(cfg, n))
                                                      for n in ("q_feat", "k_feat", "v_feat", "inner")}})


def _oracle_cfg(cfg):
    ocfg = {"variant": cfg.variant, "width": cfg.width, "block_size": cfg.block_size, "backend": cfg.backend,
            **{n: getattr(cfg, n) for n in ("w_q", "w_k", "w_v", "w_out")}}
    for n in ("q_feat", "k_feat", "v_feat", "inner"):
        g = getattr(cfg, n)
        fs = []
        for f in g.filters:
            if isinstance(f, hy.ExplicitFilter):
                fs.append(("explicit", f.taps))
            elif isinstance(f, hy.RegularizedFilter):
                fs.append(("regularized", f.taps_hat, f.decay_rate, f.base))
            else:
                fs.append(("implicit", f.residues, f.poles, f.length))
        ocfg[n] = {"channels": g.channels, "group_size": g.group_size, "filters": fs}
    return ocfg


@pytest.mark.parametrize("variant,B,D,L,kw", [
    ("MR", 2, 256, 2048, {"inner_len": 128, "block_size": 128}),
    ("MR", 1, 256, 1024, {"inner_len": 300, "block_size": 128, "group_size": 4}),
    ("SE", 1, 128, 1024, {}),
    ("LI", 1, 128, 4096, {"backend": "fft"}),
])
def test_operator_fused_projection_vs_oracle(variant, B, D, L, kw):
    """HyenaOperator with the fused projection route (qkv_fused: hy_qkv_feat_gemm, then the
    K-block / implicit conv gated by fq) against the fp64 oracle, and against the default route."""
    cfg = _rounded_cfg(variant, D, L, 3, **kw)
    x = _bf16(np.stack([hy.make_rng(4, stream=b).standard_normal((D, L)) for b in range(B)]))
    op = hy.HyenaOperator(cfg, torch.bfloat16)
    xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
    base = op.forward(xt).float().cpu().numpy()
    op.qkv_fused = True
    assert op.qkv_fused_eligible(L)
    y = op.forward(xt).float().cpu().numpy()
    ocfg = _oracle_cfg(cfg)
    for b in range(B):
        want = oracle.hyena_forward(x[b], ocfg)
        assert oracle.rel_err(y[b], want) < 1e-2, b
        assert oracle.rel_err(y[b], base[b]) < 1e-2, b


@pytest.mark.parametrize("B,D,L", [(3, 128, 256), (1, 640, 768), (2, 512, 2304), (1, 1024, 256)])
def test_qkv_feat_gemm_shapes(B, D, L):
    """Edge shapes: one time tile per sequence, an odd batch, odd 128-row tile counts (single-CTA
    path: D = 128, 640), CTA pairs with a ragged time-tile count (L = 2304 = 9 tiles)."""
    x, w, taps = _case(B, D, L, 7, 11 + D)
    fq, u = ops.qkv_feat_gemm(x, ops.qkv_weight_permute(w), taps)
    for b in {0, B - 1}:
        for c in {0, D // 2 + 1, D - 1}:
            wq, wu = _want(x, w, taps, b, c)
            assert oracle.rel_err(fq[b, c].double().cpu().numpy(), wq) < 1e-2, (b, c)
            assert oracle.rel_err(u[b, c].double().cpu().numpy(), wu) < 1e-2, (b, c)
