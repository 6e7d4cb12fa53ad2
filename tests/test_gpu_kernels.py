"""GPU parity of the sm_100a kernels against the oracle and the reference golden vectors.

Tolerances (rel_err = ||a-b||_inf / max(||b||_inf, 1), testing.py:57-62):
  fp64 path: 1e-12; fp32 path: 1e-5 (north star); bf16 path: 1e-2 against the
  fp64 oracle run on bf16-representable inputs and parameters (north star).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import ops

from .helpers import explicit_bank_from_taps, load, product_groups_from_taps

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5, "bf16": 1e-2}


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


# ---------------------------------------------------------------- direct conv


def test_direct_conv_golden():
    z = load("direct_conv")
    for i in range(3):
        x = hy.SeqTensor(np.asarray(z[f"hand{i}.x"], dtype=np.float64))
        got = hy.direct_causal_conv(x, product_groups_from_taps(z[f"hand{i}.taps"], 1))
        assert np.array_equal(got.data, z[f"hand{i}.y"]), i
    for i in range(int(z["n_rand"])):
        x = hy.SeqTensor(z[f"rand{i}.x"])
        got = hy.direct_causal_conv(x, product_groups_from_taps(z[f"rand{i}.taps"], int(z[f"rand{i}.gs"])))
        assert got.dtype == x.dtype
        assert oracle.rel_err(got.data, z[f"rand{i}.y"]) < TOL[x.dtype], i


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (3, 2, 1023, 7), (2, 5, 1025, 33), (1, 4, 3000, 300),
                                   (2, 3, 8, 20), (4, 2, 4097, 14)])
def test_causal_conv_batched_vs_oracle(dtype, shape):
    B, C, L, lh = shape
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal((B, C, L))
    taps = rng.standard_normal((C, lh)) / np.sqrt(lh)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    y = ops.causal_conv(dev(x, tdt), dev(taps, tdt), 1).cpu().numpy()
    for b in range(B):
        want = oracle.direct_causal_conv(x[b], explicit_bank_from_taps(taps, 1))
        assert oracle.rel_err(y[b], want) < TOL[dtype]


def test_causal_conv_bf16_unaligned_length():
    rng = np.random.default_rng(5)
    x = bf16_round(rng.standard_normal((2, 3, 1001)))
    taps = bf16_round(rng.standard_normal((3, 9)) / 3)
    y = ops.causal_conv(dev(x, torch.bfloat16), dev(taps), 1).float().cpu().numpy()
    for b in range(2):
        want = oracle.direct_causal_conv(x[b], explicit_bank_from_taps(taps, 1))
        assert oracle.rel_err(y[b], want) < TOL["bf16"]


def test_direct_conv_properties():
    rng = hy.make_rng(11)
    taps = rng.standard_normal((3, 5))
    groups = product_groups_from_taps(taps, 1)
    x = rng.standard_normal((3, 40))
    bumped = x.copy()
    bumped[:, 25] += 1.0
    a = hy.direct_causal_conv(hy.SeqTensor(x), groups).data[:, :25]
    b = hy.direct_causal_conv(hy.SeqTensor(bumped), groups).data[:, :25]
    assert np.array_equal(a, b)  # causality
    x2 = rng.standard_normal((3, 40))
    lhs = hy.direct_causal_conv(hy.SeqTensor(3.0 * x - 0.5 * x2), groups).data
    rhs = 3.0 * hy.direct_causal_conv(hy.SeqTensor(x), groups).data - 0.5 * hy.direct_causal_conv(
        hy.SeqTensor(x2), groups).data
    assert np.max(np.abs(lhs - rhs)) < 1e-12  # linearity
    # grouping == replication
    t4 = rng.standard_normal(4)
    x6 = rng.standard_normal((6, 30))
    by_group = hy.GroupSpec(6, 3, (hy.ExplicitFilter(t4),) * 2)
    repl = hy.GroupSpec(6, 1, (hy.ExplicitFilter(t4),) * 6)
    assert np.array_equal(hy.direct_causal_conv(hy.SeqTensor(x6), by_group).data,
                          hy.direct_causal_conv(hy.SeqTensor(x6), repl).data)


# ---------------------------------------------------------------- blocked API


def test_two_stage_block_chunk_golden():
    z = load("blockconv")
    for i in range(int(z["n_ts"])):
        v = hy.SeqTensor(z[f"ts{i}.v"])
        q = hy.SeqTensor(z[f"ts{i}.q"]) if f"ts{i}.q" in z else None
        k = hy.SeqTensor(z[f"ts{i}.k"]) if f"ts{i}.k" in z else None
        groups = product_groups_from_taps(z[f"ts{i}.taps"], int(z[f"ts{i}.gs"]))
        got = hy.two_stage_forward(v, groups, int(z[f"ts{i}.lb"]), q=q, k=k)
        assert oracle.rel_err(got.data, z[f"ts{i}.y"]) < TOL[v.dtype], i
    v = hy.SeqTensor(z["mixed.v"])
    got = hy.two_stage_forward(v, product_groups_from_taps(z["mixed.taps"], int(z["mixed.gs"])), 8)
    assert oracle.rel_err(got.data, z["mixed.y"]) < 1e-12
    for i in range(int(z["n_bk"])):
        got = hy.block_conv(hy.SeqTensor(z[f"bk{i}.x"]), product_groups_from_taps(z[f"bk{i}.taps"], int(z[f"bk{i}.gs"])),
                            int(z[f"bk{i}.lb"]))
        assert oracle.rel_err(got.data, z[f"bk{i}.y"]) < 1e-12, i
    got = hy.chunk_parallel_forward(hy.SeqTensor(z["cp.x"]), z["cp.taps"], 8)
    assert oracle.rel_err(got.data, z["cp.y"]) < 1e-12


def test_multiply_counter_both_factors():
    rng = hy.make_rng(49)
    counter = hy.MultiplyCounter()
    x = hy.SeqTensor(rng.standard_normal((4, 64)))
    groups = hy.GroupSpec(4, 2, tuple(hy.ExplicitFilter(rng.standard_normal(9)) for _ in range(2)))
    hy.two_stage_forward(x, groups, 8, counter=counter)
    assert counter.multiplies == 2 * 8 * 8 * 4 * 8


# ---------------------------------------------------------------- tcgen05 two-stage (bf16)


@pytest.mark.parametrize("B,C,L,lh,gs,gated", [
    (1, 2, 4096, 128, 1, True),
    (2, 3, 8192, 129, 1, True),
    (1, 4, 1024, 7, 2, True),
    (3, 2, 5000, 100, 1, False),
    (1, 2, 128, 128, 1, True),
    (2, 4, 12296, 64, 4, True),
    (1, 1, 8, 3, 1, True),
])
def test_two_stage_tcgen05_vs_oracle(B, C, L, lh, gs, gated):
    rng = np.random.default_rng(B * 1000 + C * 100 + L + lh)
    G = C // gs
    taps = bf16_round(rng.standard_normal((G, lh)) / np.sqrt(lh))
    v = bf16_round(rng.standard_normal((B, C, L)))
    q = bf16_round(rng.standard_normal((B, C, L))) if gated else None
    k = bf16_round(rng.standard_normal((B, C, L))) if gated else None
    y = ops.two_stage(dev(v, torch.bfloat16), dev(taps), gs,
                      q=None if q is None else dev(q, torch.bfloat16),
                      k=None if k is None else dev(k, torch.bfloat16)).float().cpu().numpy()
    bank = explicit_bank_from_taps(taps, gs)
    for b in range(B):
        want = oracle.two_stage_forward(v[b], bank, 128, q=None if q is None else q[b],
                                        k=None if k is None else k[b])
        err = oracle.rel_err(y[b], want)
        assert err < TOL["bf16"], (b, err)


def test_two_stage_tcgen05_decay_fused():
    rng = np.random.default_rng(7)
    C, L, lh = 4, 4096, 128
    taps_hat = bf16_round(rng.standard_normal((C, lh)) / np.sqrt(lh))
    rates = np.linspace(0.01, 2.0, C)
    v, q, k = (bf16_round(rng.standard_normal((1, C, L))) for _ in range(3))
    y = ops.two_stage(dev(v, torch.bfloat16), dev(taps_hat), 1, q=dev(q, torch.bfloat16), k=dev(k, torch.bfloat16),
                      decay=dev(rates * np.log2(2.0))).float().cpu().numpy()
    bank = {"channels": C, "group_size": 1,
            "filters": [("regularized", taps_hat[c], float(rates[c]), 2.0) for c in range(C)]}
    want = oracle.two_stage_forward(v[0], bank, 128, q=q[0], k=k[0])
    assert oracle.rel_err(y[0], want) < TOL["bf16"]


def test_two_stage_tcgen05_known_answers():
    # delta filter: y = q * k * v exactly in bf16 arithmetic (one nonzero tap)
    rng = np.random.default_rng(3)
    C, L = 2, 4096
    taps = np.zeros((C, 128))
    taps[:, 0] = 1.0
    v = bf16_round(rng.standard_normal((1, C, L)))
    y = ops.two_stage(dev(v, torch.bfloat16), dev(taps), 1).float().cpu().numpy()
    assert np.array_equal(y, v)
    # pure delay by 128 (exercises T1 only): y[t] = v[t-128]
    taps = np.zeros((C, 129))
    taps[:, 128] = 1.0
    y = ops.two_stage(dev(v, torch.bfloat16), dev(taps), 1).float().cpu().numpy()
    want = np.zeros_like(v)
    want[..., 128:] = v[..., :-128]
    assert np.array_equal(y, want)
    with pytest.raises(hy.TwoStageIneligibleError):
        ops.two_stage(dev(v, torch.bfloat16), dev(np.ones((C, 130))), 1)


# ---------------------------------------------------------------- fused mixers


def _mixer_oracle(proj, feat, inner_bank):
    """q * conv_inner(k * v) from raw projections (hyena.py:170-186), fp64."""
    B, C3, L = proj.shape
    C = C3 // 3
    out = np.empty((B, C, L))
    for b in range(B):
        q, k, v = (oracle.direct_causal_conv(proj[b, i * C:(i + 1) * C], explicit_bank_from_taps(feat[i], 1))
                   for i in range(3))
        out[b] = q * oracle.direct_causal_conv(k * v, inner_bank)
    return out


@pytest.mark.parametrize("B,C,L,lhf,lh,gs", [(2, 4, 8192, 7, 128, 1), (1, 3, 4104, 14, 129, 1),
                                            (1, 4, 4096, 3, 7, 2), (2, 2, 136, 7, 100, 1)])
def test_mr_mixer_tcgen05_vs_oracle(B, C, L, lhf, lh, gs):
    rng = np.random.default_rng(L + lh)
    proj = bf16_round(rng.standard_normal((B, 3 * C, L)))
    feat = bf16_round(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    taps = bf16_round(rng.standard_normal((C // gs, lh)) / np.sqrt(lh))
    y = ops.hyena_mixer(dev(proj, torch.bfloat16), dev(feat), dev(taps), gs).float().cpu().numpy()
    want = _mixer_oracle(proj, feat, explicit_bank_from_taps(taps, gs))
    assert oracle.rel_err(y, want) < TOL["bf16"]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,C,L,lhf,lh,gs", [(1, 4, 4096, 7, 7, 1), (2, 3, 1000, 14, 14, 3), (1, 2, 2049, 3, 16, 1),
                                            (3, 5, 1000, 7, 7, 5), (2, 6, 2056, 8, 5, 2), (2, 64, 8192, 7, 7, 1),
                                            (1, 8, 264, 4, 8, 4)])
def test_se_mixer_vs_oracle(dtype, B, C, L, lhf, lh, gs):
    rng = np.random.default_rng(L + lh + lhf)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    proj = rnd(rng.standard_normal((B, 3 * C, L)))
    feat = rnd(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    taps = rnd(rng.standard_normal((C // gs, lh)) / np.sqrt(lh))
    y = ops.hyena_mixer(dev(proj, tdt), dev(feat), dev(taps), gs, se_only=True).float().cpu().numpy()
    want = _mixer_oracle(np.asarray(dev(proj, tdt).double().cpu()), feat, explicit_bank_from_taps(taps, gs))
    assert oracle.rel_err(y, want) < TOL[dtype]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_se_mixer_decay_vs_oracle(dtype):
    """Regularised inner taps (core.py:146): the decay 2^(-rate*log2(base)*t) applied in-kernel."""
    B, C, L, lhf, lh = 2, 16, 6144, 7, 7
    rng = np.random.default_rng(7)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    rnd = (lambda a: a) if dtype == "f32" else bf16_round
    proj = rnd(rng.standard_normal((B, 3 * C, L)))
    feat = rnd(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    taps = rnd(rng.standard_normal((C, lh)) / np.sqrt(lh))
    dec = np.linspace(0.01, 2.0, C).astype(np.float32)
    y = ops.hyena_mixer(dev(proj, tdt), dev(feat), dev(taps), 1, decay=dev(dec), se_only=True).float().cpu().numpy()
    eff = taps * np.exp2(-dec.astype(np.float64)[:, None] * np.arange(lh)[None, :])
    want = _mixer_oracle(np.asarray(dev(proj, tdt).double().cpu()), feat, explicit_bank_from_taps(eff, 1))
    assert oracle.rel_err(y, want) < TOL[dtype]


def test_halo_correction_matches_overlap_scheme():
    rng = np.random.default_rng(9)
    C, L, lh = 3, 64, 9
    taps = rng.standard_normal((C, lh))
    halo = rng.standard_normal((C, lh - 1))
    local = rng.standard_normal((C, L))
    bank = explicit_bank_from_taps(taps, 1)
    want = oracle.direct_causal_conv(np.concatenate([halo, local], axis=1), bank)[:, lh - 1:]
    y = ops.causal_conv(dev(local, torch.float64), dev(taps, torch.float64), 1)
    ops.halo_correction(dev(halo, torch.float64), y, dev(taps, torch.float64), 1)
    assert oracle.rel_err(y.cpu().numpy(), want) < 1e-12


# ---------------------------------------------------------------- implicit long filter (LI)


def _implicit_bank(residues, poles, L, gs):
    return {"channels": residues.shape[0] * gs, "group_size": gs,
            "filters": [("implicit", r, p, L) for r, p in zip(residues, poles)]}


@pytest.mark.parametrize("B,C,L,gs,gated", [(1, 4, 8192, 1, True), (2, 3, 12288, 1, True), (1, 4, 4096, 2, False),
                                            (1, 2, 5000 // 8 * 8, 1, True)])
def test_li_conv_vs_oracle(B, C, L, gs, gated):
    rng = np.random.default_rng(L + C)
    G = C // gs
    poles = rng.uniform(-0.95, 0.95, (G, 8))
    poles[0, :4] = [0.999, -0.999, 1.0, -1.0]  # the long tail (SURVEY 7.4 hard part 5)
    poles[-1, 0] = 0.0
    residues = rng.standard_normal((G, 8)) / 8
    v = bf16_round(rng.standard_normal((B, C, L)))
    q = bf16_round(rng.standard_normal((B, C, L))) if gated else None
    k = bf16_round(rng.standard_normal((B, C, L))) if gated else None
    y = ops.li_conv(dev(v, torch.bfloat16), dev(residues), dev(poles), gs,
                    q=None if q is None else dev(q, torch.bfloat16),
                    k=None if k is None else dev(k, torch.bfloat16)).float().cpu().numpy()
    taps = oracle.bank_taps_per_channel(_implicit_bank(residues, poles, L, gs))
    for b in range(B):
        u = v[b] * (k[b] if gated else 1.0)
        want = oracle.fft_conv(u, taps) * (q[b] if gated else 1.0)
        err = oracle.rel_err(y[b], want)
        assert err < TOL["bf16"], (b, err)


def test_li_conv_many_sequences_per_cta():
    # more sequences than SMs: each CTA walks several sequences and must reset the carried state
    rng = np.random.default_rng(11)
    C, L = 320, 4096
    poles = rng.uniform(-0.99, 0.99, (C, 8))
    residues = rng.standard_normal((C, 8)) / 8
    v = bf16_round(rng.standard_normal((1, C, L)))
    y = ops.li_conv(dev(v, torch.bfloat16), dev(residues), dev(poles), 1).float().cpu().numpy()
    taps = oracle.bank_taps_per_channel(_implicit_bank(residues, poles, L, 1))
    sel = [0, 1, 147, 148, 149, 200, 319]
    want = oracle.fft_conv(v[0][sel], taps[sel])
    assert oracle.rel_err(y[0][sel], want) < TOL["bf16"]


@pytest.mark.parametrize("m", [8192, 4096])
def test_li_conv_segmented_equals_natural(m):
    # the all-to-all buffer layout (n_seg, C, seg_len): row c = buf[0, c] | buf[1, c] | ...
    # (segments of 8192: the 64-chunk kernel; 4096: the 32-chunk kernel's segmented mode)
    rng = np.random.default_rng(12)
    n, C = 3, 40
    poles = dev(rng.uniform(-0.99, 0.99, (C, 8)))
    residues = dev(rng.standard_normal((C, 8)) / 8)
    v = dev(bf16_round(rng.standard_normal((C, n * m))), torch.bfloat16)
    want = ops.li_conv(v, residues, poles, 1)
    buf = v.reshape(C, n, m).permute(1, 0, 2).contiguous()
    got = ops.li_conv_segmented(buf, residues, poles, 1)
    assert torch.equal(got.permute(1, 0, 2).reshape(C, n * m), want)
    with pytest.raises(ValueError):
        ops.li_conv_segmented(buf[..., :1000].contiguous(), residues, poles, 1)


@pytest.mark.parametrize("dtype,B,C,L,lh,gs,gated", [
    ("f32", 1, 3, 4096, 4096, 1, True),        # N = 8192: one row pass, N1 = 2
    ("f32", 2, 4, 1000, 777, 2, True),         # ragged L, lh < L, groups
    ("f32", 1, 2, 20000, 20000, 1, False),     # N = 65536: N1 = 16 column transforms
    ("f32", 1, 2, 5, 3, 1, True),              # tiny: N padded to 16
    ("bf16", 1, 3, 16384, 16384, 1, True),
    # register four-step path (fft_fast.cu): N = 8192 * N1 for N1 = 2 .. 32
    ("f32", 2, 4, 9000, 100, 2, True),          # N = 16384, N1 = 2, groups, batch
    ("bf16", 1, 2, 70000, 5000, 1, True),       # N = 131072, N1 = 16, lh < L
    ("f32", 1, 2, 131072, 131072, 1, True),     # N = 262144, N1 = 32 (config C3 size)
    # even group sizes: two channels per complex transform (real / imaginary parts)
    ("bf16", 1, 8, 131072, 131072, 4, True),
    ("f32", 2, 6, 16384, 16384, 2, False),
    # per-channel filters in pairs: the mirror-bin product (rows k1 and N1 - k1 in one CTA)
    ("f32", 2, 6, 9000, 9000, 1, True),          # N1 = 2: both rows self-paired
    ("f32", 1, 4, 65536, 30000, 1, False),       # N1 = 16
])
def test_fft_conv_vs_oracle(dtype, B, C, L, lh, gs, gated):
    # fp32 complex FFT conv (fft.py:128-145 semantics: zero-padded, truncated to L) vs the
    # float64 radix-2 oracle; fp32 tolerance 1e-5, bf16 1e-2
    rng = np.random.default_rng(L + lh)
    G = C // gs
    taps = rng.standard_normal((G, lh)) / np.sqrt(lh)
    rnd = bf16_round if dtype == "bf16" else (lambda a: a.astype(np.float32).astype(np.float64))
    v = rnd(rng.standard_normal((B, C, L)))
    q = rnd(rng.standard_normal((B, C, L))) if gated else None
    k = rnd(rng.standard_normal((B, C, L))) if gated else None
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    y = ops.fft_conv(dev(v, tdt), dev(taps), gs, q=None if q is None else dev(q, tdt),
                     k=None if k is None else dev(k, tdt)).double().cpu().numpy()
    per_ch = np.repeat(taps, gs, axis=0)
    for b in range(B):
        u = v[b] * (k[b] if gated else 1.0)
        want = oracle.fft_conv(u, per_ch) * (q[b] if gated else 1.0)
        err = oracle.rel_err(y[b], want)
        assert err < TOL[dtype], (b, err)


def test_fft_conv_errors():
    v = torch.zeros((1, 2, 64), device="cuda")
    with pytest.raises(ValueError):
        ops.fft_conv(v, torch.zeros((2, 65), device="cuda"), 1)  # lh > L


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_featurize_fwd_with_history(dtype):
    """hy_featurize_fwd: (u, fq) from the projections; with rhist = the 8 steps before t = 0 it
    equals the second half of a full-sequence run (the context-parallel halo property)."""
    B, C, L, lhf = 2, 6, 4096, 7
    rng = np.random.default_rng(21)
    rnd = bf16_round if dtype == "bf16" else (lambda a: np.asarray(a, dtype=np.float32).astype(np.float64))
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    proj = rnd(rng.standard_normal((B, 3 * C, L)))
    feat = rnd(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    u, fq = ops.featurize(dev(proj, tdt), dev(feat))
    want_u = np.empty((B, C, L))
    want_q = np.empty((B, C, L))
    for b in range(B):
        fqq, fk, fv = (oracle.direct_causal_conv(proj[b, i * C:(i + 1) * C], explicit_bank_from_taps(feat[i], 1))
                       for i in range(3))
        want_u[b], want_q[b] = fk * fv, fqq
    tol = TOL[dtype]
    assert oracle.rel_err(u.double().cpu().numpy(), want_u) < tol
    assert oracle.rel_err(fq.double().cpu().numpy(), want_q) < tol
    pd = dev(proj, tdt)
    for cut in (2048, 1000, 256):
        u2, fq2 = ops.featurize(pd[..., cut:].contiguous(), dev(feat), rhist=pd[..., cut - 8:cut].contiguous())
        assert torch.equal(u2, u[..., cut:]) and torch.equal(fq2, fq[..., cut:]), cut


@pytest.mark.parametrize("dtype,B,C,L,lh,gs", [
    ("f32", 2, 4, 12000, 9000, 2),
    ("bf16", 1, 3, 131072, 131072, 1),
])
def test_fft_conv_cached_spectrum(dtype, B, C, L, lh, gs):
    """hy_fft_spectrum once + hy_fft_conv_spec_fwd (the filter transform as a parameter
    transform) against the float64 oracle; sizes outside 2^14 <= N <= 2^18 report None."""
    rng = np.random.default_rng(L + 7)
    G = C // gs
    taps = rng.standard_normal((G, lh)) / np.sqrt(lh)
    rnd = bf16_round if dtype == "bf16" else (lambda a: a.astype(np.float32).astype(np.float64))
    v, q, k = (rnd(rng.standard_normal((B, C, L))) for _ in range(3))
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    spec = ops.fft_spectrum(dev(taps), L)
    assert spec is not None
    y = ops.fft_conv(dev(v, tdt), None, gs, q=dev(q, tdt), k=dev(k, tdt), spectrum=spec).double().cpu().numpy()
    per_ch = np.repeat(taps, gs, axis=0)
    for b in range(B):
        want = oracle.fft_conv(v[b] * k[b], per_ch) * q[b]
        assert oracle.rel_err(y[b], want) < TOL[dtype], b
    assert ops.fft_spectrum(dev(taps[:, :100]), 4000) is None  # N = 8192: not cached


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B,C,L,lh,gs,gates", [
    (1, 3, 8, 7, 1, ""),            # one partial chunk
    (2, 5, 264, 7, 1, ""),          # a full chunk + a partial one
    (3, 64, 4096, 7, 2, ""),        # many warps start mid-row (warm-up chunk)
    (1, 300, 2048, 5, 3, "kq"),     # gated, groups
    (2, 7, 1000, 8, 1, "k"),        # ungated output gate only on k
    (1, 9, 520, 3, 1, "q"),
])
def test_fir_stream_vs_oracle(dtype, B, C, L, lh, gs, gates):
    """Kernel F as a TMA-fed chunk stream (lh <= 8, L % 8 == 0): y = [q *] conv([k *] v)
    against the float64 oracle, and equal to the tiled kernel (HY_FIR_TILED) within rounding."""
    import os
    rng = np.random.default_rng(L * 7 + lh)
    G = C // gs
    taps = rng.standard_normal((G, lh)) / np.sqrt(lh)
    rnd = bf16_round if dtype == "bf16" else (lambda a: a.astype(np.float32).astype(np.float64))
    v = rnd(rng.standard_normal((B, C, L)))
    k = rnd(rng.standard_normal((B, C, L))) if "k" in gates else None
    q = rnd(rng.standard_normal((B, C, L))) if "q" in gates else None
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    args = dict(q=None if q is None else dev(q, tdt), k=None if k is None else dev(k, tdt))
    y = ops.gated_conv(dev(v, tdt), dev(taps), gs, **args)
    per_ch = np.repeat(taps, gs, axis=0)
    yn = y.double().cpu().numpy()
    for b in range(B):
        u = v[b] * (k[b] if k is not None else 1.0)
        want = oracle.direct_causal_conv(u, explicit_bank_from_taps(per_ch, 1)) * (q[b] if q is not None else 1.0)
        assert oracle.rel_err(yn[b], want) < TOL[dtype], b
    os.environ["HY_FIR_TILED"] = "1"
    try:
        y2 = ops.gated_conv(dev(v, tdt), dev(taps), gs, **args)
    finally:
        os.environ.pop("HY_FIR_TILED")
    assert float((y.double() - y2.double()).abs().max()) <= (2e-2 if dtype == "bf16" else 1e-5) * max(
        1.0, float(y2.double().abs().max()))


@pytest.mark.parametrize("shape", [(2, 48, 256), (1, 7, 13), (3, 16, 4104)])
def test_split3_cat_kernel_exact(shape):
    """hy_split3_cat writes [X1; X2; X0; X1; X0] with X0 + X1 + X2 == x exactly (blas.py)."""
    from paper_2503_01868_b200 import blas
    g = torch.Generator(device="cuda").manual_seed(sum(shape))
    x = torch.randn(shape, device="cuda", generator=g) * torch.logspace(-8, 8, shape[-1], device="cuda")
    s = blas.split3_act(x)
    B, K, N = shape
    parts = s.cat.view(B, 5, K, N)
    x0, x1, x2 = blas.split3(x)  # the eager restatement
    assert torch.equal(parts[:, 0], x1) and torch.equal(parts[:, 1], x2) and torch.equal(parts[:, 2], x0)
    assert torch.equal(parts[:, 3], x1) and torch.equal(parts[:, 4], x0) and torch.equal(s[0], x0)
    assert torch.equal(x0.double() + x1.double() + x2.double(), x.double())


def test_split3_matmul_fp32_parity():
    """fp32 GEMM through the split kernel + six bf16 products vs fp64, within the fp32 bar."""
    from paper_2503_01868_b200 import blas
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn((384, 4096), device="cuda", generator=g) / 64
    x = torch.randn((2, 4096, 512), device="cuda", generator=g)
    got = blas.matmul_split3(blas.split3_weight(a), blas.split3_act(x))
    want = torch.matmul(a.double(), x.double())
    err = float((got.double() - want).abs().max() / max(1.0, float(want.abs().max())))
    assert err < 1e-5, err


# ---------------------------------------------------------------- modal scan (LI at reference precision)


@pytest.mark.parametrize("dtype,B,C,L,gs,np_,gated", [
    ("f32", 1, 4, 8192, 1, 8, True),
    ("f32", 2, 6, 1000, 2, 3, True),        # ragged L (scalar loads), groups, 3 poles
    ("f32", 1, 3, 1, 1, 8, False),          # L = 1
    ("f32", 1, 5, 131072, 1, 8, True),      # config C3's length, tail poles
    ("f32", 1, 4, 20000, 1, 12, True),      # 12 poles: two mode blocks
    ("f32", 1, 2, 9000, 1, 64, False),      # 64 poles
    ("f64", 2, 3, 5000, 1, 8, True),
    ("f64", 1, 2, 131072, 1, 8, False),
    ("bf16", 1, 4, 12288, 1, 16, True),     # > 8 poles (the tcgen05 kernel's limit)
    ("bf16", 1, 3, 1001, 3, 8, True),       # L % 8 != 0
])
def test_li_scan_vs_oracle(dtype, B, C, L, gs, np_, gated):
    """hy_li_scan_fwd against the fp64 oracle's fft_conv on the materialised implicit filter
    (fft.py:128-145, core.py:147-151): fp32 1e-5 and bf16 1e-2 (north star), fp64 1e-10."""
    rng = np.random.default_rng(L + C + np_)
    G = C // gs
    poles = rng.uniform(-0.95, 0.95, (G, np_))
    poles[0, :min(np_, 5)] = [1.0, -1.0, 0.9999, -0.9999, 0.0][:min(np_, 5)]
    residues = rng.standard_normal((G, np_)) / np_
    rnd = {"f32": lambda a: a.astype(np.float32).astype(np.float64), "f64": lambda a: a, "bf16": bf16_round}[dtype]
    tdt = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}[dtype]
    v = rnd(rng.standard_normal((B, C, L)))
    q = rnd(rng.standard_normal((B, C, L))) if gated else None
    k = rnd(rng.standard_normal((B, C, L))) if gated else None
    y = ops.li_scan(dev(v, tdt), torch.from_numpy(residues), torch.from_numpy(poles), gs,
                    q=None if q is None else dev(q, tdt), k=None if k is None else dev(k, tdt)).double().cpu().numpy()
    taps = oracle.bank_taps_per_channel(_implicit_bank(residues, poles, L, gs))
    tol = {"f32": 1e-5, "f64": 1e-10, "bf16": 1e-2}[dtype]
    for b in range(B):
        u = v[b] * (k[b] if gated else 1.0)
        want = oracle.fft_conv(u, taps) * (q[b] if gated else 1.0)
        err = oracle.rel_err(y[b], want)
        assert err < tol, (b, err)


def test_li_scan_many_rows_and_errors():
    """More rows than resident CTAs (each CTA re-initialises its tables and carries per row);
    argument errors map to the reference's exception types."""
    rng = np.random.default_rng(3)
    C, L = 700, 4100
    poles = rng.uniform(-0.99, 0.99, (C, 8))
    residues = rng.standard_normal((C, 8)) / 8
    v = rng.standard_normal((1, C, L)).astype(np.float32).astype(np.float64)
    y = ops.li_scan(dev(v), torch.from_numpy(residues), torch.from_numpy(poles), 1).double().cpu().numpy()
    sel = [0, 1, 295, 296, 597, 699]
    taps = oracle.bank_taps_per_channel(_implicit_bank(residues[sel], poles[sel], L, 1))
    assert oracle.rel_err(y[0][sel], oracle.fft_conv(v[0][sel], taps)) < 1e-5
    with pytest.raises(NotImplementedError):
        ops.li_scan(dev(v[:, :4]), torch.zeros((4, 65), dtype=torch.float64), torch.zeros((4, 65), dtype=torch.float64))
    with pytest.raises(ValueError):
        ops.li_scan(dev(v[:, :4]), torch.zeros((3, 8), dtype=torch.float64), torch.zeros((3, 8), dtype=torch.float64))


@pytest.mark.parametrize("dtype,B,C,L,lhf,np_", [("f32", 2, 5, 8192, 7, 8), ("f32", 1, 3, 1000, 4, 3),
                                                 ("bf16", 1, 4, 16384, 7, 12), ("f64", 1, 3, 3000, 8, 8),
                                                 ("f32", 1, 2, 131072, 7, 8)])
def test_li_scan_mixer_vs_oracle(dtype, B, C, L, lhf, np_):
    """Fused LI mixer on the modal scan (featurizers + gates + implicit conv from the projections)
    against the oracle's featurizer convs and fft_conv."""
    rng = np.random.default_rng(L + lhf + np_)
    poles = rng.uniform(-0.95, 0.95, (C, np_))
    poles[0, :3] = [1.0, -0.9999, 0.0]
    residues = rng.standard_normal((C, np_)) / np_
    rnd = {"f32": lambda a: a.astype(np.float32).astype(np.float64), "f64": lambda a: a, "bf16": bf16_round}[dtype]
    tdt = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}[dtype]
    proj = rnd(rng.standard_normal((B, 3 * C, L)))
    feat = rnd(rng.standard_normal((3, C, lhf)) / np.sqrt(lhf))
    y = ops.li_scan_mixer(dev(proj, tdt), dev(feat, torch.float64 if dtype == "f64" else torch.float32),
                          torch.from_numpy(residues), torch.from_numpy(poles), 1)
    y = y.double().cpu().numpy()
    taps = oracle.bank_taps_per_channel(_implicit_bank(residues, poles, L, 1))
    tol = {"f32": 1e-5, "f64": 1e-10, "bf16": 1e-2}[dtype]
    for b in range(B):
        fq, fk, fv = (oracle.direct_causal_conv(proj[b, i * C:(i + 1) * C], explicit_bank_from_taps(feat[i], 1))
                      for i in range(3))
        want = fq * oracle.fft_conv(fk * fv, taps)
        err = oracle.rel_err(y[b], want)
        assert err < tol, (b, err)


# ---------------------------------------------------------------- K-block tcgen05 conv (lh > lb + 1)


@pytest.mark.parametrize("B,C,L,lh,gs,gated,decay", [
    (1, 4, 8192, 130, 1, False, False),     # K = 2 at the kernel's LB = 128
    (2, 3, 8192, 257, 1, True, False),      # K = 2 / 3 boundary
    (1, 4, 12296, 385, 2, True, True),      # K = 3, groups, partial tile, decay
    (1, 2, 4096, 513, 1, False, False),     # K = 4 (the maximum)
    (1, 2, 600, 300, 1, False, False),      # shorter than one tile
    (4, 1024, 8192, 200, 1, True, True),    # many tiles and filter groups per CTA (C2-like walk)
    (1, 4096, 4096, 300, 16, False, True),  # a factor rebuild every 16 tiles, 28 groups per CTA
])
def test_block_conv_tcgen05_vs_oracle(B, C, L, lh, gs, gated, decay):
    """hy_block_conv_fwd (K + 1 accumulating tcgen05 MMAs over row-shifted U views) against the
    oracle's block_conv / two_stage semantics (blockconv.py:103-121, 182-220), bf16 bar 1e-2."""
    rng = np.random.default_rng(L + lh + C)
    G = C // gs
    taps = bf16_round(rng.standard_normal((G, lh)) / np.sqrt(lh))
    rates = np.linspace(0.001, 0.02, G) if decay else None
    sel = sorted({0, C - 1, C // 2, 147 % C, 148 % C, 149 % C}) if C > 64 else list(range(C))
    g = torch.Generator(device="cuda").manual_seed(L + lh)
    v, q, k = (torch.randn((B, C, L), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    y = ops.block_conv(v, dev(taps), gs, q=q if gated else None, k=k if gated else None,
                       decay=None if rates is None else dev(rates * np.log2(2.0))).double().cpu().numpy()
    vh, qh, kh = (t.double().cpu().numpy() for t in (v, q, k))
    worst = 0.0
    for c in sel:
        spec = ("regularized", taps[c // gs], float(rates[c // gs]), 2.0) if decay else ("explicit", taps[c // gs])
        bank = {"channels": 1, "group_size": 1, "filters": [spec]}
        for b in range(B):
            u = vh[b, c:c + 1] * (kh[b, c:c + 1] if gated else 1.0)
            want = oracle.block_conv(u, bank, 16) * (qh[b, c:c + 1] if gated else 1.0)
            worst = max(worst, oracle.rel_err(y[b, c:c + 1], want))
    assert worst < TOL["bf16"], worst


def test_block_conv_tcgen05_golden_and_known_answers():
    """The reference's block_conv goldens (bk*, any block size) through the bf16 K-block kernel,
    plus exact known answers: a delay of 400 steps (factor T_3 only) and a delta."""
    z = load("blockconv")
    for i in range(int(z["n_bk"])):
        x = bf16_round(z[f"bk{i}.x"])
        taps = z[f"bk{i}.taps"]
        gs = int(z[f"bk{i}.gs"])
        y = ops.block_conv(dev(x, torch.bfloat16), dev(taps), gs).double().cpu().numpy()
        want = oracle.block_conv(x, explicit_bank_from_taps(taps, gs), int(z[f"bk{i}.lb"]))
        assert oracle.rel_err(y, want) < TOL["bf16"], i
        assert oracle.rel_err(y, z[f"bk{i}.y"]) < 2e-2, i  # golden on the unrounded input
    rng = np.random.default_rng(4)
    v = bf16_round(rng.standard_normal((1, 3, 8192)))
    taps = np.zeros((3, 401))
    taps[:, 400] = 1.0
    y = ops.block_conv(dev(v, torch.bfloat16), dev(taps), 1).float().cpu().numpy()
    want = np.zeros_like(v)
    want[..., 400:] = v[..., :-400]
    assert np.array_equal(y, want)
    taps = np.zeros((3, 513))
    taps[:, 0] = 1.0
    y = ops.block_conv(dev(v, torch.bfloat16), dev(taps), 1).float().cpu().numpy()
    assert np.array_equal(y, v)
    with pytest.raises(NotImplementedError):
        ops.block_conv(dev(v, torch.bfloat16), dev(np.ones((3, 514))), 1)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("n", [1, 7, 4096, 100003])
def test_gate_mul(dtype, n):
    """hy_gate_mul (the CP LI layer's q gate): bitwise the rounding of the fp32 / fp64 product."""
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(n, device="cuda", generator=g).to(dtype)
    b = torch.randn(n, device="cuda", generator=g).to(dtype)
    want = (a.double() * b.double()).to(dtype) if dtype != torch.float64 else a * b
    assert torch.equal(ops.gate_mul(a, b), want)


def test_new_kernels_edge_cases():
    """Edge shapes of this round's kernels: K-block conv with lh = 1 (only T_0), L = 1 and L < 8
    (padded rows), groups; modal scan with L = 1 and a single pole; FFT over more rows than a
    grid dimension holds."""
    rng = np.random.default_rng(17)
    for B, C, L, lh, gs in ((2, 4, 1, 1, 2), (1, 3, 5, 200, 3), (3, 2, 8, 130, 1)):
        v = bf16_round(rng.standard_normal((B, C, L)))
        taps = bf16_round(rng.standard_normal((C // gs, lh)) / np.sqrt(lh))
        y = ops.block_conv(dev(v, torch.bfloat16), dev(taps), gs).double().cpu().numpy()
        for b in range(B):
            want = oracle.block_conv(v[b], explicit_bank_from_taps(taps, gs), 16)
            assert oracle.rel_err(y[b], want) < TOL["bf16"], (B, C, L, lh)
    v = rng.standard_normal((2, 3, 1))
    y = ops.li_scan(dev(v), torch.tensor([[0.5]] * 3, dtype=torch.float64), torch.tensor([[0.9]] * 3, dtype=torch.float64))
    assert np.allclose(y.double().cpu().numpy(), 0.5 * v.astype(np.float32), rtol=1e-6)
    x = torch.randn((70000, 4), dtype=torch.complex64, device="cuda")
    got = ops.fft_c2c(x).cpu().numpy()
    want = np.fft.fft(x.cpu().numpy(), axis=-1)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-5
