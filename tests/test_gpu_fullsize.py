"""Parity at the BASELINE configs' full sizes through size-independent properties.

At C1 / C2 / C3 sizes the fp64 oracle cannot run the whole workload, so each kernel is checked
at its full benchmark size by properties that hold exactly in the device arithmetic, plus an
oracle check on channels sampled across every CTA's range:

* scaling: the mixers are cubic in the projections (y = fq * h * (fk * fv)) and the convs are
  linear, and multiplying by 2 is exact in bf16 / fp32 (products, sums, FMAs with the taps and
  the modal powers all scale by a power of two), so y(2 p) == 8 y(p) and conv(2 v) == 2 conv(v)
  must hold bitwise;
* causality: perturbing the input at time t0 must leave every output before the 128-step chunk
  that contains t0 bitwise unchanged (an output chunk never reads a later chunk's column of the
  MMAs, nor a later tile's state);
* sampled channels against the oracle (the conv is channel-separable): bf16 1e-2, fp32 1e-5.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import ops

pytestmark = pytest.mark.gpu

D = 4096


def _conv(x, h):
    return np.convolve(x, h)[: x.shape[-1]]


def _check_props(fn, inp, scale_pow, t0, tol_chans=None):
    """scaling (bitwise), causality (bitwise) of fn on inp (..., L); returns y."""
    y = fn(inp)
    y2 = fn(inp * 2)
    assert torch.equal(y2, y * (2 ** scale_pow)), "scaling by 2 is not exact"
    pert = inp.clone()
    pert[..., t0] += 3.0
    yp = fn(pert)
    c0 = t0 // 128 * 128
    assert torch.equal(yp[..., :c0], y[..., :c0]), "an output before the perturbed chunk changed"
    assert not torch.equal(yp[..., t0:], y[..., t0:])
    return y


def _sample(C):
    return sorted({0, 1, C // 3, C // 2, 2 * C // 3, C - 2, C - 1, 147, 148, 2000})


def test_mr_mixer_c2_full_size():
    """Config C2's mixer: B = 4, C = 4096, L = 8192 (1.07 GB per launch), the bench's kernel."""
    g = torch.Generator(device="cuda").manual_seed(1)
    B, L = 4, 8192
    proj = torch.randn((B, 3 * D, L), device="cuda", generator=g).to(torch.bfloat16)
    feat = (torch.randn((3, D, 7), device="cuda", generator=g) / 2.65).to(torch.bfloat16).float()
    taps = (torch.randn((D, 128), device="cuda", generator=g) / 11.3).to(torch.bfloat16).float()
    dec = torch.linspace(0.01, 2.0, D, device="cuda")
    packed = ops.feat_pack(feat)
    y = _check_props(lambda p: ops.hyena_mixer(p, feat, taps, 1, decay=dec, packed=packed), proj, 3, 5000)
    fh, th, rh = feat.double().cpu().numpy(), taps.double().cpu().numpy(), dec.double().cpu().numpy()
    for c in _sample(D):
        h = oracle.materialize(("regularized", th[c], rh[c], 2.0))
        fq, fk, fv = (_conv(proj[1, i * D + c].double().cpu().numpy(), fh[i, c]) for i in range(3))
        assert oracle.rel_err(y[1, c].double().cpu().numpy(), fq * _conv(fk * fv, h)) < 1e-2, c


def _li_modes(seed):
    rng = np.random.default_rng(seed)
    poles = rng.uniform(-0.95, 0.95, (D, 8))
    poles[0, :4] = [1.0, -1.0, 0.9999, 0.0]
    residues = rng.standard_normal((D, 8)) / 8
    return residues, poles


def test_li_mixer_c3_full_size():
    """Config C3's LI mixer: B = 1, C = 4096, L = 131072 (4.3 GB per launch)."""
    g = torch.Generator(device="cuda").manual_seed(2)
    L = 131072
    residues, poles = _li_modes(3)
    proj = torch.randn((1, 3 * D, L), device="cuda", generator=g).to(torch.bfloat16)
    feat = (torch.randn((3, D, 7), device="cuda", generator=g) / 2.65).to(torch.bfloat16).float()
    packed = ops.feat_pack(feat)
    rt, pt = torch.from_numpy(residues).float().cuda(), torch.from_numpy(poles).float().cuda()
    y = _check_props(lambda p: ops.li_mixer(p, feat, rt, pt, 1, packed=packed), proj, 3, 100003)
    fh = feat.double().cpu().numpy()
    for c in (0, 147, 2000, D - 1):
        ph = [proj[0, i * D + c].double().cpu().numpy() for i in range(3)]
        fq, fk, fv = (_conv(ph[i], fh[i, c]) for i in range(3))
        want = fq * oracle.fft_conv(fk * fv, oracle.materialize(("implicit", residues[c], poles[c], L)))
        assert oracle.rel_err(y[0, c].double().cpu().numpy(), want) < 1e-2, c


def test_li_conv_c3_full_size():
    """The ungated implicit conv (the CP slab kernel) at C3 size: linear, causal, oracle."""
    g = torch.Generator(device="cuda").manual_seed(4)
    L = 131072
    residues, poles = _li_modes(5)
    v = torch.randn((1, D, L), device="cuda", generator=g).to(torch.bfloat16)
    rt, pt = torch.from_numpy(residues).float().cuda(), torch.from_numpy(poles).float().cuda()
    y = _check_props(lambda x: ops.li_conv(x, rt, pt, 1), v, 1, 77777)
    for c in (0, 1, 1500, D - 1):
        want = oracle.fft_conv(v[0, c].double().cpu().numpy(), oracle.materialize(("implicit", residues[c], poles[c], L)))
        assert oracle.rel_err(y[0, c].double().cpu().numpy(), want) < 1e-2, c


def test_se_mixer_c1_full_size_fp32():
    """Config C1's fp32 SE mixer (B = 1, C = 4096, L = 4096): exact scaling / causality, fp32
    1e-5 on sampled channels."""
    g = torch.Generator(device="cuda").manual_seed(6)
    L = 4096
    proj = torch.randn((1, 3 * D, L), device="cuda", generator=g)
    feat = torch.randn((3, D, 7), device="cuda", generator=g) / 2.65
    taps = torch.randn((D, 7), device="cuda", generator=g) / 2.65
    y = _check_props(lambda p: ops.hyena_mixer(p, feat, taps, 1), proj, 3, 3000)
    fh, th = feat.double().cpu().numpy(), taps.double().cpu().numpy()
    for c in _sample(D):
        ph = [proj[0, i * D + c].double().cpu().numpy() for i in range(3)]
        fq, fk, fv = (_conv(ph[i], fh[i, c]) for i in range(3))
        assert oracle.rel_err(y[0, c].double().cpu().numpy(), fq * _conv(fk * fv, th[c])) < 1e-5, c


def test_block_conv_full_size():
    """K-block conv (lh = 300, K = 3) at the C2 activation size, gated: exact scaling (cubic in
    the three inputs scaled together) and causality."""
    g = torch.Generator(device="cuda").manual_seed(7)
    B, L = 4, 8192
    v, q, k = (torch.randn((B, D, L), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    taps = torch.randn((D, 300), device="cuda", generator=g) / 17
    y = ops.block_conv(v, taps, 1, q=q, k=k)
    assert torch.equal(ops.block_conv(2 * v, taps, 1, q=2 * q, k=2 * k), 8 * y)
    vp = v.clone()
    vp[..., 6000] += 3.0
    yp = ops.block_conv(vp, taps, 1, q=q, k=k)
    assert torch.equal(yp[..., :5888], y[..., :5888])
    th = taps.double().cpu().numpy()
    for c in (0, 2047, D - 1):
        qh = q[2, c].double().cpu().numpy()
        want = qh * _conv(k[2, c].double().cpu().numpy() * v[2, c].double().cpu().numpy(), th[c])
        assert oracle.rel_err(y[2, c].double().cpu().numpy(), want) < 1e-2, c


def test_mr_operator_c2_full_size_properties():
    """The whole C2 operator (cuBLAS projections + mixer), B = 4, L = 8192, D = 4096: scaling the
    input by 2 scales y by 8 bitwise (bf16 GEMMs with fp32 accumulation scale exactly), and the
    operator is causal (projections are per time step)."""
    cfg = hy.make_hyena_config("MR", D, hy.make_rng(0), inner_len=128, block_size=128)
    op = hy.HyenaOperator(cfg, torch.bfloat16)
    g = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn((4, D, 8192), device="cuda", generator=g).to(torch.bfloat16)
    _check_props(op.forward, x, 3, 4321)
