"""CPU tests of the host-side API mirror: seeded builders, validation and errors,
factor utilities — everything that does not launch a kernel."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import blockconv as bc

from .helpers import load


def test_builders_match_reference_draws():
    z = load("builders")
    kws = (("SE", {}), ("MR", {"group_size": 2}), ("LI", {"seq_len": 32, "n_poles": 4}))
    for i, (variant, kw) in enumerate(kws):
        cfg = hy.make_hyena_config(variant, 4, hy.make_rng(1000 + i), **kw)
        for name in ("w_q", "w_k", "w_v", "w_out"):
            assert np.array_equal(getattr(cfg, name), z[f"b{i}.{name}"])
        for name in ("q_feat", "k_feat", "v_feat", "inner"):
            assert np.array_equal(getattr(cfg, name).materialized(), z[f"b{i}.{name}.materialized"])
    spec = hy.make_layout(("SE", "MR"), 2, 4, hy.make_rng(1010), seq_len=16)
    for i, cfg in enumerate(spec.layers):
        assert cfg.variant == str(z[f"lay{i}.variant"])
        assert np.array_equal(cfg.w_out, z[f"lay{i}.w_out"])
        assert np.array_equal(cfg.inner.materialized(), z[f"lay{i}.inner.materialized"])


def test_spill_and_factors_match_reference():
    cases = {(1, 3): 0, (3, 3): 1, (4, 3): 1, (5, 3): 2, (7, 3): 2, (9, 2): 4}
    for (lh, lb), want in cases.items():
        assert hy.spill_count(lh, lb) == want
    z = load("blockconv")
    f = hy.build_factors(z["factors.h"], 3)
    assert np.array_equal(f.blocks, z["factors.blocks"])
    assert f.spill_count == 1
    rng = hy.make_rng(42)
    for lh, lb, length in ((1, 4, 12), (5, 4, 16), (9, 4, 20), (6, 5, 17)):
        taps = rng.standard_normal(lh)
        assert np.array_equal(hy.assemble_toeplitz(hy.build_factors(taps, lb), length),
                              hy.full_toeplitz(taps, length))
    with pytest.raises(ValueError):
        hy.build_factors([1.0], 0)
    assert hy.two_stage_flops(1024, 64, 128) == 16777216


def test_seqtensor_and_filter_validation():
    with pytest.raises(ValueError):
        hy.SeqTensor(np.zeros(3))
    with pytest.raises(ValueError):
        hy.SeqTensor(np.array([[np.nan]]))
    with pytest.raises(ValueError):
        hy.SeqTensor(np.zeros((1, 2)), dtype="f16")
    s = hy.SeqTensor(np.zeros((2, 3), dtype=np.float32))
    assert s.dtype == "f32" and s.channels == 2 and s.length == 3
    assert not s.data.flags.writeable
    with pytest.raises(ValueError):
        hy.RegularizedFilter(np.ones(3), 0.5, base=1.0)
    with pytest.raises(ValueError):
        hy.RegularizedFilter(np.ones(3), -0.1)
    with pytest.raises(ValueError):
        hy.ImplicitFilter(np.ones(2), np.array([0.5, 1.5]), 8)
    with pytest.raises(TypeError):
        hy.materialize_filter(object())
    with pytest.raises(ValueError):
        hy.GroupSpec(4, 3, ())
    with pytest.raises(ValueError):
        hy.GroupSpec(4, 2, (hy.ExplicitFilter(np.ones(2)), hy.ExplicitFilter(np.ones(3))))
    g = hy.uniform_groups(4, [1.0, 2.0])
    assert g.n_groups == 1 and g.filter_len == 2


def test_materialize_matches_reference():
    z = load("filters")
    got = hy.materialize_filter(hy.RegularizedFilter(z["reg.taps_hat"], float(z["reg.rate"]), float(z["reg.base"])))
    assert np.array_equal(got, z["reg.y"])
    got = hy.materialize_filter(hy.ImplicitFilter(z["imp.residues"], z["imp.poles"], int(z["imp.length"])))
    assert np.array_equal(got, z["imp.y"])


def test_config_validation():
    rng = hy.make_rng(63)
    with pytest.raises(ValueError):
        hy.make_hyena_config("SE", 2, rng, inner_len=15)
    hy.make_hyena_config("SE", 2, rng, inner_len=14)
    with pytest.raises(ValueError):
        hy.make_hyena_config("SE", 2, rng, featurizer_len=15)
    with pytest.raises(ValueError):
        hy.make_hyena_config("XX", 2, rng)
    cfg = hy.make_hyena_config("MR", 2, rng, inner_len=6)
    se_bank = hy.GroupSpec(2, 2, (hy.ExplicitFilter(np.array([1.0])),))
    with pytest.raises(ValueError):
        hy.HyenaConfig(**{**cfg.__dict__, "inner": se_bank})
    with pytest.raises(ValueError):
        hy.HyenaConfig(**{**cfg.__dict__, "backend": "nope"})
    with pytest.raises(ValueError):
        hy.HyenaConfig(**{**cfg.__dict__, "w_q": np.zeros((3, 3))})
    with pytest.raises(ValueError):
        hy.make_inner_bank("LI", 2, 1, rng)


def test_input_checks_before_device():
    # shape errors are raised host-side, before any device work
    rng = hy.make_rng(67)
    cfg = hy.make_hyena_config("SE", 4, rng)
    with pytest.raises(ValueError):
        hy.hyena_forward(hy.SeqTensor(np.zeros((3, 16))), cfg)
    li = hy.make_hyena_config("LI", 2, rng, seq_len=16)
    with pytest.raises(ValueError):
        hy.hyena_forward(hy.SeqTensor(np.zeros((2, 17))), li)
    groups = hy.GroupSpec(2, 1, (hy.ExplicitFilter(np.ones(10)),) * 2)
    with pytest.raises(bc.TwoStageIneligibleError):
        hy.two_stage_forward(hy.SeqTensor(np.zeros((2, 32))), groups, 8)
    with pytest.raises(ValueError):
        hy.two_stage_forward(hy.SeqTensor(np.zeros((2, 32))), hy.GroupSpec(2, 1, (hy.ExplicitFilter(np.ones(3)),) * 2),
                             8, q=hy.SeqTensor(np.zeros((2, 31))))
    with pytest.raises(ValueError):
        hy.direct_causal_conv(hy.SeqTensor(np.zeros((3, 8))), hy.uniform_groups(4, [1.0]))


def test_layout_validation():
    rng = hy.make_rng(80)
    se = hy.make_hyena_config("SE", 4, rng)
    mr = hy.make_hyena_config("MR", 4, rng, inner_len=8)
    with pytest.raises(ValueError):
        hy.LayoutSpec(("SE", "MR"), 1, (mr, se))
    with pytest.raises(ValueError):
        hy.LayoutSpec(("SE",), 2, (se,))
    with pytest.raises(ValueError):
        hy.LayoutSpec((), 1, ())
    spec = hy.LayoutSpec(("SE", "MR"), 1, (se, mr))
    assert hy.build_layout(spec, residual=True).residual


def test_multiply_counter_model():
    counter = hy.MultiplyCounter()
    counter.add_matmul(8, 8, 32)
    assert counter.multiplies == 2048
    assert oracle.two_stage_flops(64, 8, 4) == 2 * 8 * 8 * 4 * 8


def test_backward_validation_before_device():
    """Backward entry points reject bad contexts / shapes with the reference's ValueError before
    any device work (blockconv.py:230-234, hyena.py:252-256), and the parameter traversal is
    host logic (hyena.py:291-319)."""
    with pytest.raises(ValueError):
        hy.two_stage_backward(object(), np.ones((1, 4)))
    with pytest.raises(ValueError):
        hy.hyena_backward(object(), np.ones((1, 4)))
    cfg = hy.make_hyena_config("LI", 4, hy.make_rng(3), seq_len=16, n_poles=2)
    paths = [p for p, _ in hy.iter_params(cfg)]
    assert paths[:4] == [("w_q",), ("w_k",), ("w_v",), ("w_out",)]
    assert ("inner", 0, "residues") in paths and ("inner", 3, "poles") in paths
    assert len(paths) == 4 + 3 * 4 + 2 * 4
    g = hy.HyenaGrads(dx=None, dw_q=np.ones(1), dw_k=(np.zeros(1), np.ones(2)), dw_v=None, dw_out=None,
                      filters={"inner": [{"residues": np.full(2, 3.0)}]})
    assert hy.grad_for_path(g, ("w_k", "right")).shape == (2,)
    assert hy.grad_for_path(g, ("inner", 0, "residues"))[0] == 3.0
