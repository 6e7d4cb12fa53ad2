"""GPU parity of the backward kernels (hy_causal_conv_bwd, hy_li_param_grad) against the
oracle restatement of the reference backward and the reference-generated golden vectors.

Tolerances (rel_err, testing.py:57-62): fp64 1e-12; fp32 1e-5; bf16 1e-2 against the fp64
oracle on bf16-representable inputs (north star)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from oracle import backward as ob
from paper_2503_01868_b200 import ops

from .helpers import load

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5, "bf16": 1e-2}
TDT = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def test_conv_bwd_golden_f64():
    z = load("backward")
    for n in range(int(z["n_cg"])):
        p = f"cg{n}"
        gs = int(z[f"{p}.gs"])
        dx, dt = ops.causal_conv_bwd(dev(z[f"{p}.dy"]), dev(z[f"{p}.x"]), dev(z[f"{p}.taps"]), gs)
        assert oracle.rel_err(dx.cpu().numpy(), z[f"{p}.dx"]) < TOL["f64"], p
        assert oracle.rel_err(dt.cpu().numpy(), z[f"{p}.dtaps"]) < TOL["f64"], p


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
@pytest.mark.parametrize("B,C,L,lh,gs", [(1, 4, 4096, 7, 1), (3, 6, 1000, 5, 2), (2, 4, 8192, 128, 1),
                                         (1, 3, 2051, 129, 3), (2, 2, 777, 1, 1), (1, 2, 3000, 2048, 2),
                                         (4, 8, 64, 100, 4)])
def test_conv_bwd_vs_oracle(dtype, B, C, L, lh, gs):
    rng = np.random.default_rng(B * 1000 + L + lh)
    rnd = bf16_round if dtype == "bf16" else (lambda a: a)
    dy = rnd(rng.standard_normal((B, C, L)))
    x = rnd(rng.standard_normal((B, C, L)))
    taps = rnd(rng.standard_normal((C // gs, lh)) / np.sqrt(lh))
    if dtype == "f32":
        dy, x = dy.astype(np.float32), x.astype(np.float32)
    tt = torch.float64 if dtype == "f64" else torch.float32
    dx, dt = ops.causal_conv_bwd(dev(dy, TDT[dtype]), dev(x, TDT[dtype]), dev(taps, tt), gs)
    bank = oracle.explicit_bank(C, gs, taps)
    want_dx = np.stack([ob.causal_conv_input_grad(dy[b], np.repeat(taps, gs, axis=0)) for b in range(B)])
    want_dt = sum(ob.causal_conv_taps_grad(dy[b], x[b], bank) for b in range(B))
    assert oracle.rel_err(dx.double().cpu().numpy(), want_dx) < TOL[dtype]
    assert oracle.rel_err(dt.double().cpu().numpy(), want_dt) < TOL[dtype]


def test_conv_bwd_partial_outputs_and_errors():
    rng = np.random.default_rng(3)
    dy = dev(rng.standard_normal((2, 4, 300)), torch.float32)
    x = dev(rng.standard_normal((2, 4, 300)), torch.float32)
    taps = dev(rng.standard_normal((4, 9)), torch.float32)
    dx_only, none = ops.causal_conv_bwd(dy, None, taps, 1, want_dtaps=False)
    assert none is None
    dx_both, dt_both = ops.causal_conv_bwd(dy, x, taps, 1)
    assert torch.equal(dx_only, dx_both)
    none, dt_only = ops.causal_conv_bwd(dy, x, 9, 1, want_dx=False)
    assert none is None and torch.equal(dt_only, dt_both)  # deterministic reduction
    with pytest.raises(NotImplementedError):
        ops.causal_conv_bwd(dy, x, dev(np.zeros((4, 2049)), torch.float32), 1)
    with pytest.raises(ValueError):
        ops.causal_conv_bwd(dy, x, taps, 3)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,C,L,npoles,gs,near_one", [(1, 4, 256, 8, 1, False), (2, 6, 1000, 3, 2, False),
                                                      (1, 2, 4096, 8, 1, True), (3, 4, 77, 1, 4, False)])
def test_li_param_grad_vs_oracle(dtype, B, C, L, npoles, gs, near_one):
    rng = np.random.default_rng(L + npoles)
    rnd = bf16_round if dtype == "bf16" else (lambda a: np.asarray(a, dtype=np.float32).astype(np.float64))
    dc = rnd(rng.standard_normal((B, C, L)))
    u = rnd(rng.standard_normal((B, C, L)))
    G = C // gs
    res = rnd(rng.standard_normal((G, npoles)) / npoles)
    poles = rnd(rng.uniform(0.99, 1.0, (G, npoles)) if near_one else rng.uniform(-0.95, 0.95, (G, npoles)))
    poles[0, 0] = 0.0  # 0 ** 0 = 1 (core.py:147-151)
    d_res, d_pole = ops.li_param_grad(dev(dc, TDT[dtype]), dev(u, TDT[dtype]), dev(res, torch.float32),
                                      dev(poles, torch.float32), gs)
    bank = {"channels": C, "group_size": gs, "filters": [("implicit", res[g], poles[g], L) for g in range(G)]}
    dtaps = sum(ob.causal_conv_taps_grad(dc[b], u[b], bank) for b in range(B))
    want = [ob.filter_param_grads(bank["filters"][g], dtaps[g]) for g in range(G)]
    want_res = np.stack([w["residues"] for w in want])
    want_pole = np.stack([w["poles"] for w in want])
    tol = TOL[dtype] if not near_one else 5 * TOL[dtype]
    assert oracle.rel_err(d_res.double().cpu().numpy(), want_res) < tol
    assert oracle.rel_err(d_pole.double().cpu().numpy(), want_pole) < tol


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,C,L,lhf", [(2, 4, 4096, 7), (1, 3, 1000, 8), (3, 2, 248, 7), (1, 5, 256, 3),
                                       (2, 2, 8, 7), (2, 64, 2056, 7), (1, 1, 504, 1)])
def test_featurizer_bwd_vs_oracle(dtype, B, C, L, lhf):
    """hy_featurizer_bwd = _feat_backward for q, k, v (hyena.py:234-247) with the gate products
    dq = g * c, dk = du * fv, dv = du * fk (hyena.py:262-270)."""
    rng = np.random.default_rng(L * 7 + lhf + C)
    rnd = bf16_round if dtype == "bf16" else (lambda a: np.asarray(a, dtype=np.float32).astype(np.float64))
    proj = rnd(rng.standard_normal((B, 3 * C, L)))
    g, cc, du = (rnd(rng.standard_normal((B, C, L))) for _ in range(3))
    feat = rnd(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    dproj, dfeat = ops.featurizer_bwd(dev(proj, TDT[dtype]), dev(g, TDT[dtype]), dev(cc, TDT[dtype]),
                                      dev(du, TDT[dtype]), dev(feat, torch.float32))
    want_dp = np.empty_like(proj)
    want_df = np.zeros((3, C, lhf))
    for b in range(B):
        pq, pk, pv = (proj[b, i * C:(i + 1) * C] for i in range(3))
        fk = oracle.direct_causal_conv(pk, oracle.explicit_bank(C, 1, feat[1]))
        fv = oracle.direct_causal_conv(pv, oracle.explicit_bank(C, 1, feat[2]))
        for i, (dfx, px) in enumerate(((g[b] * cc[b], pq), (du[b] * fv, pk), (du[b] * fk, pv))):
            want_dp[b, i * C:(i + 1) * C] = ob.causal_conv_input_grad(dfx, feat[i])
            want_df[i] += ob.causal_conv_taps_grad(dfx, px, oracle.explicit_bank(C, 1, feat[i]))
    tol = TOL[dtype]
    assert oracle.rel_err(dproj.double().cpu().numpy(), want_dp) < tol
    assert oracle.rel_err(dfeat.double().cpu().numpy(), want_df) < (1e-4 if dtype == "f32" else tol)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_mixer_bwd_prep_and_reversed_du(dtype):
    """hy_mixer_bwd_prep (u = fk*fv, dc = g*fq, dc reversed) and hy_featurizer_bwd reading du
    time-reversed equal the natural-order results."""
    B, C, L, lhf = 2, 6, 2056, 7
    rng = np.random.default_rng(11)
    rnd = bf16_round if dtype == "bf16" else (lambda a: np.asarray(a, dtype=np.float32).astype(np.float64))
    proj = rnd(rng.standard_normal((B, 3 * C, L)))
    g, cc, du = (rnd(rng.standard_normal((B, C, L))) for _ in range(3))
    feat = rnd(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    t = TDT[dtype]
    u, dc, dcr = ops.mixer_bwd_prep(dev(proj, t), dev(g, t), dev(feat, torch.float32), reversed_dc=True)
    want_u = np.empty((B, C, L))
    want_dc = np.empty((B, C, L))
    for b in range(B):
        fq, fk, fv = (oracle.direct_causal_conv(proj[b, i * C:(i + 1) * C], oracle.explicit_bank(C, 1, feat[i]))
                      for i in range(3))
        want_u[b], want_dc[b] = fk * fv, g[b] * fq
    assert oracle.rel_err(u.double().cpu().numpy(), want_u) < TOL[dtype]
    assert oracle.rel_err(dc.double().cpu().numpy(), want_dc) < TOL[dtype]
    assert torch.equal(torch.flip(dc, dims=[-1]), dcr)
    a = ops.featurizer_bwd(dev(proj, t), dev(g, t), dev(cc, t), dev(du, t), dev(feat, torch.float32))
    r = ops.featurizer_bwd(dev(proj, t), dev(g, t), dev(cc, t), torch.flip(dev(du, t), dims=[-1]).contiguous(),
                           dev(feat, torch.float32), du_reversed=True)
    assert torch.equal(a[0], r[0])
    assert torch.allclose(a[1], r[1], rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("B,C,L,lh,gs", [(1, 4, 8192, 128, 1), (2, 3, 8192, 129, 3), (1, 2, 1000, 128, 1),
                                         (3, 4, 16384 + 136, 100, 2), (1, 300, 256, 7, 1), (2, 2, 128, 128, 1)])
def test_two_stage_taps_grad_tcgen05_vs_oracle(B, C, L, lh, gs):
    """hy_two_stage_taps_grad (tcgen05 chunk outer products + diagonal scatter) equals the
    reference's two-pass filter gradient (blockconv.py:246-262) = causal_conv_taps_grad."""
    rng = np.random.default_rng(L + lh + C)
    dc = bf16_round(rng.standard_normal((B, C, L)))
    u = bf16_round(rng.standard_normal((B, C, L)))
    got = ops.two_stage_taps_grad(dev(dc, torch.bfloat16), dev(u, torch.bfloat16), lh, gs)
    bank = oracle.explicit_bank(C, gs, np.zeros((C // gs, lh)))
    want = sum(ob.causal_conv_taps_grad(dc[b], u[b], bank) for b in range(B))
    assert oracle.rel_err(got.double().cpu().numpy(), want) < 1e-5
