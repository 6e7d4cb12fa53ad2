"""Pin the CPU oracle against golden vectors produced by the reference itself.

These run on CPU only (no GPU, no product compute). The oracle may only be
trusted as the checker for the CUDA path once every fixture here matches.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import cpsim as ocp

from .helpers import explicit_bank_from_taps, load, oracle_cfg


def test_direct_conv_golden():
    z = load("direct_conv")
    for i in range(3):
        got = oracle.direct_causal_conv(np.asarray(z[f"hand{i}.x"], dtype=np.float64),
                                        explicit_bank_from_taps(z[f"hand{i}.taps"], 1))
        assert np.array_equal(got, z[f"hand{i}.y"])
    for i in range(int(z["n_rand"])):
        x = z[f"rand{i}.x"]
        got = oracle.direct_causal_conv(x, explicit_bank_from_taps(z[f"rand{i}.taps"], int(z[f"rand{i}.gs"])))
        assert got.dtype == x.dtype
        assert np.array_equal(got, z[f"rand{i}.y"]), i


def test_factors_and_two_stage_golden():
    z = load("blockconv")
    assert np.array_equal(oracle.build_factors(z["factors.h"], 3), z["factors.blocks"])
    for i in range(int(z["n_ts"])):
        bank = explicit_bank_from_taps(z[f"ts{i}.taps"], int(z[f"ts{i}.gs"]))
        got = oracle.two_stage_forward(z[f"ts{i}.v"], bank, int(z[f"ts{i}.lb"]),
                                       q=z.get(f"ts{i}.q"), k=z.get(f"ts{i}.k"))
        assert oracle.rel_err(got, z[f"ts{i}.y"]) < 1e-13, i
    bank = explicit_bank_from_taps(z["mixed.taps"], int(z["mixed.gs"]))
    assert oracle.rel_err(oracle.two_stage_forward(z["mixed.v"], bank, 8), z["mixed.y"]) < 1e-13
    for i in range(int(z["n_bk"])):
        bank = explicit_bank_from_taps(z[f"bk{i}.taps"], int(z[f"bk{i}.gs"]))
        got = oracle.block_conv(z[f"bk{i}.x"], bank, int(z[f"bk{i}.lb"]))
        assert oracle.rel_err(got, z[f"bk{i}.y"]) < 1e-13, i
    got = oracle.chunk_parallel_forward(z["cp.x"], z["cp.taps"], 8)
    assert oracle.rel_err(got, z["cp.y"]) < 1e-13
    assert oracle.two_stage_flops(1024, 64, 128) == int(z["flops"]) == 16777216


def test_fft_golden():
    z = load("fft")
    assert list(oracle.bit_reversal_indices(8)) == list(z["bitrev8"]) == [0, 4, 2, 6, 1, 5, 3, 7]
    assert np.max(np.abs(oracle.fft(z["fft.x"]) - z["fft.y"])) < 1e-12
    for i in range(int(z["n_fc"])):
        got = oracle.fft_conv(z[f"fc{i}.x"], z[f"fc{i}.taps"])
        assert oracle.rel_err(got, z[f"fc{i}.y"]) < 1e-13, i


def test_filters_golden():
    z = load("filters")
    spec = ("regularized", z["reg.taps_hat"], float(z["reg.rate"]), float(z["reg.base"]))
    assert np.array_equal(oracle.materialize(spec), z["reg.y"])
    spec = ("implicit", z["imp.residues"], z["imp.poles"], int(z["imp.length"]))
    assert np.array_equal(oracle.materialize(spec), z["imp.y"])


def test_hyena_golden():
    z = load("hyena")
    for i in range(int(z["n_h"])):
        cfg = oracle_cfg(z, f"h{i}.cfg")
        got = oracle.hyena_forward(z[f"h{i}.x"], cfg)
        assert got.dtype == z[f"h{i}.y"].dtype
        tol = 1e-6 if got.dtype == np.float32 else 1e-12
        assert oracle.rel_err(got, z[f"h{i}.y"]) < tol, (i, z[f"h{i}.args"])
    got = oracle.hyena_forward(z["ident.x"], oracle.identity_config(width=3))
    assert np.array_equal(got, z["ident.y"])


def test_layout_golden():
    z = load("layout")
    layers = [oracle_cfg(z, f"layer{i}") for i in range(int(z["n_layers"]))]
    for residual in (0, 1):
        for dtype in ("f32", "f64"):
            got = oracle.layout_forward(z[f"{residual}.{dtype}.x"], layers, residual=bool(residual))
            tol = 1e-6 if dtype == "f32" else 1e-12
            assert oracle.rel_err(got, z[f"{residual}.{dtype}.y"]) < tol


def test_builders_golden():
    z = load("builders")
    kws = (("SE", {}), ("MR", {"group_size": 2}), ("LI", {"seq_len": 32, "n_poles": 4}))
    for i, (variant, kw) in enumerate(kws):
        cfg = oracle.make_hyena_config(variant, 4, oracle.make_rng(1000 + i), **kw)
        want = oracle_cfg(z, f"b{i}")
        for name in ("w_q", "w_k", "w_v", "w_out"):
            assert np.array_equal(cfg[name], want[name])
        for name in ("q_feat", "k_feat", "v_feat", "inner"):
            assert np.array_equal(oracle.bank_taps(cfg[name]), oracle.bank_taps(want[name]))


def test_cpsim_golden():
    z = load("cpsim")
    for i in range(int(z["n_cp"])):
        scheme, n_ranks, d, dg, length, lh, n_pipe, layout, name = [str(a) for a in z[f"cp{i}.args"]]
        n_ranks, dg, n_pipe = int(n_ranks), int(dg), int(n_pipe)
        bank = explicit_bank_from_taps(z[f"cp{i}.taps"], dg)
        tally = ocp.Tally(n_ranks)
        xs = ocp.shard(z[f"cp{i}.x"], n_ranks, layout)
        if scheme.startswith("p2p"):
            ys = ocp.p2p_conv(xs, bank, tally, overlapped=(scheme == "p2p_ov"))
        else:
            ys = ocp.a2a_conv(xs, bank, tally, n_pipe=n_pipe, layout=layout)
        for r in range(n_ranks):
            assert np.max(np.abs(ys[r] - z[f"cp{i}.shard{r}"])) < 1e-12, (i, r)
        assert np.max(np.abs(ocp.gather(ys, layout) - z[f"cp{i}.y"])) < 1e-12
        assert tally.elements.get(name, 0) == int(z[f"cp{i}.elements"]), i
        assert tally.messages.get(name, 0) == int(z[f"cp{i}.messages"]), i
        assert tally.rounds.get(name, 0) == int(z[f"cp{i}.rounds"]), i
        assert [tally.filter_elements[r] for r in range(n_ranks)] == list(z[f"cp{i}.filter_elements"])


def test_two_stage_ineligible():
    bank = explicit_bank_from_taps(np.ones((1, 10)), 1)
    with pytest.raises(oracle.TwoStageIneligibleError):
        oracle.two_stage_forward(np.ones((1, 32)), bank, 8)
