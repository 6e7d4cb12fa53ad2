"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (the reference is importable read-only there):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz. The GPU box never runs this (it has no
/root/reference); tests only read the committed .npz files. Every case is
built from the reference's own seeded builders (make_rng / make_hyena_config /
testing.random_*), so the inputs are bit-reproducible.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from convhybrid import blockconv as bc  # noqa: E402
from convhybrid import cpsim, hyena  # noqa: E402
from convhybrid import fft as fftmod  # noqa: E402
from convhybrid.core import (  # noqa: E402
    ExplicitFilter,
    GroupSpec,
    ImplicitFilter,
    RegularizedFilter,
    SeqTensor,
    direct_causal_conv,
    materialize_filter,
    uniform_groups,
)
from convhybrid.rand import make_rng  # noqa: E402
from convhybrid.testing import random_explicit_groups, random_mixed_groups, random_seq  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def bank_arrays(prefix: str, g: GroupSpec) -> dict:
    """Serialize a GroupSpec (any filter kind, one kind per bank) to flat arrays."""
    out = {f"{prefix}.channels": g.channels, f"{prefix}.group_size": g.group_size}
    f0 = g.filters[0]
    kinds = {type(f) for f in g.filters}
    if len(kinds) > 1:
        out[f"{prefix}.kind"] = "mixed"
        out[f"{prefix}.taps"] = g.materialized()
        return out
    if isinstance(f0, ExplicitFilter):
        out[f"{prefix}.kind"] = "explicit"
        out[f"{prefix}.taps"] = np.stack([f.taps for f in g.filters])
    elif isinstance(f0, RegularizedFilter):
        out[f"{prefix}.kind"] = "regularized"
        out[f"{prefix}.taps_hat"] = np.stack([f.taps_hat for f in g.filters])
        out[f"{prefix}.rate"] = np.array([f.decay_rate for f in g.filters])
        out[f"{prefix}.base"] = np.array([f.base for f in g.filters])
    else:
        out[f"{prefix}.kind"] = "implicit"
        out[f"{prefix}.residues"] = np.stack([f.residues for f in g.filters])
        out[f"{prefix}.poles"] = np.stack([f.poles for f in g.filters])
        out[f"{prefix}.length"] = f0.length
    out[f"{prefix}.materialized"] = g.materialized()
    return out


def cfg_arrays(prefix: str, cfg: hyena.HyenaConfig) -> dict:
    out = {f"{prefix}.variant": cfg.variant, f"{prefix}.width": cfg.width,
           f"{prefix}.block_size": cfg.block_size, f"{prefix}.backend": cfg.backend}
    for name in ("w_q", "w_k", "w_v", "w_out"):
        out[f"{prefix}.{name}"] = hyena.projection_dense(getattr(cfg, name))
    for name in ("q_feat", "k_feat", "v_feat", "inner"):
        out.update(bank_arrays(f"{prefix}.{name}", getattr(cfg, name)))
    return out


def save(name: str, cases: dict) -> None:
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **{k: np.asarray(v) for k, v in cases.items()})
    print(f"wrote {path} ({len(cases)} arrays)")


def gen_direct() -> None:
    c = {}
    # reference hand values (pkg/tests/test_core.py:124-137)
    c["hand0.x"] = [[1.0, 2.0, 3.0, 4.0]]
    c["hand0.taps"] = [[1.0, 1.0]]
    c["hand0.y"] = direct_causal_conv(SeqTensor(c["hand0.x"]), uniform_groups(1, [1.0, 1.0])).data
    c["hand1.x"] = [[1.0, 2.0, 3.0, 4.0]]
    c["hand1.taps"] = [[0.0, 1.0]]
    c["hand1.y"] = direct_causal_conv(SeqTensor(c["hand1.x"]), uniform_groups(1, [0.0, 1.0])).data
    c["hand2.x"] = [[1.0, 1.0]]
    c["hand2.taps"] = [[1.0, 2.0, 3.0, 4.0]]
    c["hand2.y"] = direct_causal_conv(SeqTensor(c["hand2.x"]), uniform_groups(1, [1.0, 2.0, 3.0, 4.0])).data
    for i in range(3):
        c[f"hand{i}.gs"] = 1
    rng = make_rng(500)
    shapes = [(3, 1, 40, 5), (4, 2, 50, 6), (2, 1, 3, 9), (6, 3, 30, 4), (8, 8, 64, 14),
              (5, 1, 33, 1), (16, 1, 300, 7), (4, 2, 257, 40), (2, 1, 1000, 129), (3, 3, 4099, 7)]
    n = 0
    for dtype in ("f64", "f32"):
        for d, gs, length, lh in shapes:
            g = random_explicit_groups(rng, d, gs, lh)
            x = random_seq(rng, d, length, dtype=dtype)
            y = direct_causal_conv(x, g)
            c[f"rand{n}.x"] = x.data
            c[f"rand{n}.taps"] = g.materialized()
            c[f"rand{n}.gs"] = gs
            c[f"rand{n}.y"] = y.data
            n += 1
    c["n_rand"] = n
    save("direct_conv", c)


def gen_blockconv() -> None:
    c = {}
    rng = make_rng(510)
    # paper H0/H1 worked example (pkg/tests/test_blockconv.py:25-42)
    h = rng.standard_normal(4)
    f = bc.build_factors(h, 3)
    c["factors.h"] = h
    c["factors.blocks"] = f.blocks
    # two-stage (gated and ungated), both dtypes
    n = 0
    for dtype in ("f64", "f32"):
        for d, dg, length, lh, lb, gated in ((1, 1, 48, 3, 4, False), (4, 4, 96, 17, 16, False),
                                              (6, 2, 65, 8, 8, True), (4, 2, 40, 5, 8, True),
                                              (8, 1, 1000, 129, 128, True), (3, 1, 300, 128, 128, True),
                                              (2, 2, 2051, 100, 128, False), (5, 1, 130, 7, 16, True)):
            g = random_explicit_groups(rng, d, dg, lh)
            v = random_seq(rng, d, length, dtype)
            q = random_seq(rng, d, length, dtype) if gated else None
            k = random_seq(rng, d, length, dtype) if gated else None
            y = bc.two_stage_forward(v, g, lb, q=q, k=k)
            c[f"ts{n}.v"] = v.data
            if gated:
                c[f"ts{n}.q"] = q.data
                c[f"ts{n}.k"] = k.data
            c[f"ts{n}.taps"] = g.materialized()
            c[f"ts{n}.gs"] = dg
            c[f"ts{n}.lb"] = lb
            c[f"ts{n}.y"] = y.data
            n += 1
    c["n_ts"] = n
    # mixed filter kinds through two-stage (regularized decay in the path)
    g = random_mixed_groups(rng, 6, 2, 9)
    v = random_seq(rng, 6, 77)
    c["mixed.v"] = v.data
    c["mixed.taps"] = g.materialized()
    c["mixed.gs"] = 2
    c["mixed.y"] = bc.two_stage_forward(v, g, 8).data
    # block_conv (pkg/tests/test_blockconv.py:70-83 shapes)
    n = 0
    for d, dg, length, lh, lb in ((1, 1, 32, 4, 8), (4, 2, 100, 9, 16), (8, 4, 257, 40, 16),
                                  (2, 1, 64, 64, 8), (4, 1, 600, 300, 128)):
        g = random_explicit_groups(rng, d, dg, lh)
        x = random_seq(rng, d, length)
        c[f"bk{n}.x"] = x.data
        c[f"bk{n}.taps"] = g.materialized()
        c[f"bk{n}.gs"] = dg
        c[f"bk{n}.lb"] = lb
        c[f"bk{n}.y"] = bc.block_conv(x, g, lb).data
        n += 1
    c["n_bk"] = n
    # chunk-parallel
    taps = rng.standard_normal(9) / 3.0
    x = random_seq(rng, 5, 70)
    c["cp.x"] = x.data
    c["cp.taps"] = taps
    c["cp.y"] = bc.chunk_parallel_forward(x, taps, 8).data
    c["flops"] = bc.two_stage_flops(1024, 64, 128)
    save("blockconv", c)


def gen_fft() -> None:
    c = {}
    rng = make_rng(520)
    n = 0
    for d, length, lh in ((1, 16, 16), (3, 100, 100), (2, 64, 10), (4, 257, 257), (2, 1024, 1024),
                          (1, 5, 3)):
        x = rng.standard_normal((d, length))
        taps = rng.standard_normal((d, lh)) / np.sqrt(lh)
        c[f"fc{n}.x"] = x
        c[f"fc{n}.taps"] = taps
        c[f"fc{n}.y"] = fftmod.fft_conv(x, taps)
        n += 1
    c["n_fc"] = n
    z = rng.standard_normal(32) + 1j * rng.standard_normal(32)
    c["fft.x"] = z
    c["fft.y"] = fftmod.fft(z)
    c["bitrev8"] = fftmod.bit_reversal_indices(8)
    save("fft", c)


def gen_filters() -> None:
    c = {}
    rng = make_rng(530)
    th = rng.standard_normal(10)
    c["reg.taps_hat"] = th
    c["reg.rate"] = 0.7
    c["reg.base"] = 2.0
    c["reg.y"] = materialize_filter(RegularizedFilter(th, 0.7, 2.0))
    res = rng.standard_normal(5)
    poles = np.array([-1.0, -0.5, 0.0, 0.99, 1.0])
    c["imp.residues"] = res
    c["imp.poles"] = poles
    c["imp.length"] = 300
    c["imp.y"] = materialize_filter(ImplicitFilter(res, poles, 300))
    save("filters", c)


def gen_hyena() -> None:
    c = {}
    n = 0
    specs = [
        # (variant, width, L, group_size, inner_len, block_size, backend, dtype)
        ("SE", 8, 64, 1, None, 16, "blocked", "f32"),
        ("SE", 8, 96, 2, 9, 8, "direct", "f64"),
        ("SE", 8, 96, 2, 9, 8, "fft", "f64"),
        ("SE", 16, 200, 1, 14, 16, "blocked", "f32"),
        ("MR", 8, 256, 1, 128, 128, "blocked", "f32"),
        ("MR", 8, 300, 2, 128, 128, "blocked", "f64"),
        ("MR", 4, 64, 1, 24, 8, "blocked", "f64"),  # spill > 1 -> block_conv route
        ("MR", 8, 130, 1, 64, 16, "direct", "f32"),
        ("LI", 8, 64, 1, None, 16, "fft", "f32"),
        ("LI", 8, 256, 2, None, 16, "fft", "f64"),
        ("LI", 4, 48, 1, None, 16, "direct", "f64"),
    ]
    for variant, width, length, gs, inner_len, lb, backend, dtype in specs:
        rng = make_rng(600 + n)
        cfg = hyena.make_hyena_config(variant, width, rng, seq_len=length, group_size=gs,
                                      inner_len=inner_len, block_size=lb, backend=backend)
        x = random_seq(make_rng(700 + n), width, length, dtype)
        y = hyena.hyena_forward(x, cfg)
        c.update(cfg_arrays(f"h{n}.cfg", cfg))
        c[f"h{n}.seed"] = 600 + n
        c[f"h{n}.x"] = x.data
        c[f"h{n}.y"] = y.data
        c[f"h{n}.args"] = np.array([variant, str(width), str(length), str(gs), str(inner_len), str(lb),
                                    backend, dtype])
        n += 1
    c["n_h"] = n
    # identity collapse (pkg/tests/test_hyena.py:21-25)
    x = random_seq(make_rng(60), 3, 24)
    c["ident.x"] = x.data
    c["ident.y"] = hyena.hyena_forward(x, hyena.identity_config(width=3)).data
    save("hyena", c)


def gen_layout() -> None:
    c = {}
    width, length = 8, 64
    rng = make_rng(800)
    layers = (
        hyena.make_hyena_config("SE", width, rng, seq_len=length, block_size=16),
        hyena.make_hyena_config("MR", width, rng, seq_len=length, inner_len=32, block_size=32),
        hyena.make_hyena_config("LI", width, rng, seq_len=length, backend="fft"),
    )
    spec = hyena.LayoutSpec(("SE", "MR", "LI"), 1, layers)
    for residual in (False, True):
        for dtype in ("f32", "f64"):
            stack = hyena.build_layout(spec, residual=residual)
            x = random_seq(make_rng(801), width, length, dtype)
            c[f"{int(residual)}.{dtype}.x"] = x.data
            c[f"{int(residual)}.{dtype}.y"] = hyena.layout_forward(x, stack).data
    for i, cfg in enumerate(layers):
        c.update(cfg_arrays(f"layer{i}", cfg))
    c["n_layers"] = len(layers)
    save("layout", c)


def gen_cpsim() -> None:
    c = {}
    n = 0
    for scheme, n_ranks, d, dg, length, lh, n_pipe, layout in (
        ("p2p", 4, 8, 2, 256, 7, 1, "sequential"),
        ("p2p_ov", 4, 8, 4, 128, 9, 1, "sequential"),
        ("p2p", 2, 4, 1, 64, 1, 1, "sequential"),
        ("a2a", 4, 16, 1, 256, 9, 1, "sequential"),
        ("a2a", 4, 16, 1, 256, 9, 1, "zigzag"),
        ("a2a_pipe", 4, 16, 1, 128, 7, 2, "sequential"),
        ("a2a", 2, 8, 2, 64, 64, 1, "sequential"),
    ):
        rng = make_rng(900 + n)
        groups = random_explicit_groups(rng, d, dg, lh)
        x = random_seq(rng, d, length)
        grp = cpsim.SimGroup(n_ranks)
        xs = cpsim.shard(x, n_ranks, layout)
        if scheme == "p2p":
            ys = cpsim.p2p_conv(xs, groups, grp)
            name = "p2p_conv"
        elif scheme == "p2p_ov":
            ys = cpsim.p2p_conv_overlapped(xs, groups, grp)
            name = "p2p_conv_overlapped"
        elif scheme == "a2a":
            ys = cpsim.a2a_conv(xs, groups, grp)
            name = "a2a_conv"
        else:
            ys = cpsim.a2a_conv_pipelined(xs, groups, grp, n_pipe)
            name = "a2a_conv_pipelined"
        c[f"cp{n}.args"] = np.array([scheme, str(n_ranks), str(d), str(dg), str(length), str(lh),
                                     str(n_pipe), layout, name])
        c[f"cp{n}.x"] = x.data
        c[f"cp{n}.taps"] = groups.materialized()
        c[f"cp{n}.y"] = cpsim.gather(ys).data
        for r in range(n_ranks):
            c[f"cp{n}.shard{r}"] = ys.shards[r]
        c[f"cp{n}.elements"] = grp.total_elements(name)
        c[f"cp{n}.messages"] = grp.total_messages(name)
        c[f"cp{n}.rounds"] = grp.scheme_rounds.get(name, 0)
        c[f"cp{n}.filter_elements"] = np.array([grp.filter_elements[r] for r in range(n_ranks)])
        n += 1
    c["n_cp"] = n
    save("cpsim", c)


def gen_dfft() -> None:
    """Distributed FFT scheme (cpsim.py:537-659), cases of pkg/tests/test_cpsim.py:324-412."""
    c = {}
    for n_ranks, seed, length in ((2, 111, 16), (4, 112, 32)):
        rng = make_rng(seed)
        x = rng.standard_normal((1, length))
        spectra = cpsim.p2p_fft_forward(cpsim.shard(SeqTensor(x), n_ranks), cpsim.SimGroup(n_ranks))
        c[f"own{n_ranks}.x"] = x
        for r in range(n_ranks):
            c[f"own{n_ranks}.spec{r}"] = spectra[r]
    for n_ranks in (2, 4, 8):
        rng = make_rng(114)
        x = rng.standard_normal((2, 64))
        h = rng.standard_normal((2, 64))
        grp = cpsim.SimGroup(n_ranks)
        ys = cpsim.p2p_fft_conv(cpsim.shard(SeqTensor(x), n_ranks), cpsim.shard(SeqTensor(h), n_ranks), grp)
        c[f"conv{n_ranks}.x"] = x
        c[f"conv{n_ranks}.h"] = h
        c[f"conv{n_ranks}.y"] = cpsim.gather(ys).data
        c[f"conv{n_ranks}.elements"] = grp.total_elements("p2p_fft_conv")
        c[f"conv{n_ranks}.messages"] = grp.total_messages("p2p_fft_conv")
        c[f"conv{n_ranks}.rounds"] = grp.scheme_rounds.get("p2p_fft_conv", 0)
        c[f"conv{n_ranks}.max_resident"] = max(grp.max_resident.values())
    rng = make_rng(118)
    taps = rng.standard_normal(24) / np.sqrt(24)
    x = random_seq(rng, 2, 96)
    c["causal.taps"] = taps
    c["causal.x"] = x.data
    c["causal.y"] = cpsim.p2p_fft_causal_wrapper(x, taps, 4, cpsim.SimGroup(4)).data
    rng = make_rng(119)
    taps = rng.standard_normal(40)
    x = random_seq(rng, 1, 32)
    c["trunc.taps"] = taps
    c["trunc.x"] = x.data
    c["trunc.y"] = cpsim.p2p_fft_causal_wrapper(x, taps, 2, cpsim.SimGroup(2)).data
    save("dfft", c)


def gen_builders() -> None:
    """Raw make_hyena_config draws, to pin the product's seeded builders."""
    c = {}
    for i, (variant, kw) in enumerate((("SE", {}), ("MR", {"group_size": 2}),
                                       ("LI", {"seq_len": 32, "n_poles": 4}))):
        cfg = hyena.make_hyena_config(variant, 4, make_rng(1000 + i), **kw)
        c.update(cfg_arrays(f"b{i}", cfg))
    layout = hyena.make_layout(("SE", "MR"), 2, 4, make_rng(1010), seq_len=16)
    for i, cfg in enumerate(layout.layers):
        c.update(cfg_arrays(f"lay{i}", cfg))
    save("builders", c)


def grads_arrays(prefix: str, g: "hyena.HyenaGrads") -> dict:
    """HyenaGrads -> flat arrays: dx, dense/factored projection grads, filter leaves stacked
    over groups ({prefix}.f.{role}.{leaf} of shape (n_groups, ...))."""
    out = {f"{prefix}.dx": g.dx}
    for name in ("dw_q", "dw_k", "dw_v", "dw_out"):
        val = getattr(g, name)
        if isinstance(val, tuple):
            out[f"{prefix}.{name}.left"], out[f"{prefix}.{name}.right"] = val
        else:
            out[f"{prefix}.{name}"] = val
    for role, per_group in g.filters.items():
        for leaf in per_group[0]:
            out[f"{prefix}.f.{role}.{leaf}"] = np.stack([d[leaf] for d in per_group])
    return out


def gen_backward() -> None:
    """Reference backward passes: conv adjoints (core.py:245-268), two-stage backward
    (blockconv.py:223-264, incl. the hand example of pkg/tests/test_blockconv.py:154-160),
    operator backward per variant/backend/dtype (hyena.py:250-284), layout backward
    (hyena.py:409-417) and the sharded a2a backward (cpsim.py:440-446)."""
    from convhybrid.core import causal_conv_input_grad, causal_conv_taps_grad
    c = {}
    rng = make_rng(1100)
    n = 0
    for d, gs, length, lh in ((3, 1, 40, 5), (4, 2, 50, 6), (2, 1, 3, 9), (6, 3, 300, 7), (4, 4, 257, 40),
                              (2, 1, 1000, 129), (5, 5, 64, 1)):
        g = random_explicit_groups(rng, d, gs, lh)
        x = rng.standard_normal((d, length))
        dy = rng.standard_normal((d, length))
        c[f"cg{n}.x"], c[f"cg{n}.dy"], c[f"cg{n}.taps"], c[f"cg{n}.gs"] = x, dy, g.materialized(), gs
        c[f"cg{n}.dx"] = causal_conv_input_grad(dy, g.taps_per_channel())
        c[f"cg{n}.dtaps"] = causal_conv_taps_grad(dy, x, g)
        n += 1
    c["n_cg"] = n
    # two-stage backward: hand example, then random gated / ungated
    _, saved = bc.two_stage_forward_saved(SeqTensor([[1.0, 2.0, 3.0, 4.0]]), uniform_groups(1, [1.0, 1.0]), 2)
    hg = bc.two_stage_backward(saved, np.ones((1, 4)))
    c["hand.dtaps"], c["hand.dv"] = hg.dtaps, hg.dv
    n = 0
    for dtype in ("f64", "f32"):
        for d, dg, length, lh, lb, gated in ((4, 2, 24, 5, 4, True), (6, 3, 70, 9, 8, False),
                                              (4, 1, 300, 128, 128, True), (3, 3, 260, 129, 128, True),
                                              (2, 1, 130, 7, 16, True)):
            g = random_explicit_groups(rng, d, dg, lh)
            v = random_seq(rng, d, length, dtype)
            q = random_seq(rng, d, length, dtype) if gated else None
            k = random_seq(rng, d, length, dtype) if gated else None
            dy = rng.standard_normal((d, length))
            _, saved = bc.two_stage_forward_saved(v, g, lb, q=q, k=k)
            tg = bc.two_stage_backward(saved, dy)
            c[f"tb{n}.v"], c[f"tb{n}.dy"] = v.data, dy
            if gated:
                c[f"tb{n}.q"], c[f"tb{n}.k"] = q.data, k.data
                c[f"tb{n}.dq"], c[f"tb{n}.dk"] = tg.dq, tg.dk
            c[f"tb{n}.taps"], c[f"tb{n}.gs"], c[f"tb{n}.lb"] = g.materialized(), dg, lb
            c[f"tb{n}.dv"], c[f"tb{n}.dtaps"] = tg.dv, tg.dtaps
            n += 1
    c["n_tb"] = n
    # operator backward
    specs = [
        ("SE", 8, 64, 1, None, 16, "blocked", "f64", False),
        ("SE", 8, 96, 2, 9, 8, "direct", "f32", True),
        ("SE", 4, 40, 1, None, 16, "fft", "f64", False),
        ("MR", 8, 256, 1, 128, 128, "blocked", "f64", False),
        ("MR", 8, 300, 2, 128, 128, "blocked", "f32", False),
        ("MR", 4, 64, 1, 24, 8, "blocked", "f64", True),
        ("MR", 8, 130, 1, 64, 16, "direct", "f32", False),
        ("LI", 8, 64, 1, None, 16, "fft", "f64", False),
        ("LI", 4, 48, 2, None, 16, "direct", "f32", False),
        ("LI", 8, 256, 1, None, 16, "fft", "f64", True),
    ]
    n = 0
    for variant, width, length, gs, inner_len, lb, backend, dtype, factored in specs:
        rng = make_rng(1200 + n)
        cfg = hyena.make_hyena_config(variant, width, rng, seq_len=length, group_size=gs,
                                      inner_len=inner_len, block_size=lb, backend=backend)
        if factored:
            r = max(1, width // 2)
            cfg = dataclasses.replace(cfg, w_v=(rng.standard_normal((width, r)), rng.standard_normal((r, width))))
            c[f"hb{n}.cfg.w_v.left"], c[f"hb{n}.cfg.w_v.right"] = cfg.w_v
        x = random_seq(make_rng(1300 + n), width, length, dtype)
        dy = make_rng(1400 + n).standard_normal((width, length))
        y, saved = hyena.hyena_forward_saved(x, cfg)
        g = hyena.hyena_backward(saved, dy)
        c.update(cfg_arrays(f"hb{n}.cfg", cfg))
        c.update(grads_arrays(f"hb{n}.g", g))
        c[f"hb{n}.x"], c[f"hb{n}.dy"], c[f"hb{n}.y"] = x.data, dy, y.data
        c[f"hb{n}.args"] = np.array([variant, str(width), str(length), str(gs), str(inner_len), str(lb),
                                     backend, dtype, str(factored)])
        n += 1
    c["n_hb"] = n
    # layout backward (residual stack SE-MR-LI)
    width, length = 8, 64
    rng = make_rng(1500)
    layers = (hyena.make_hyena_config("SE", width, rng, seq_len=length, block_size=16),
              hyena.make_hyena_config("MR", width, rng, seq_len=length, inner_len=32, block_size=32),
              hyena.make_hyena_config("LI", width, rng, seq_len=length, block_size=16))
    stack = hyena.OperatorStack(layers, residual=True)
    x = random_seq(make_rng(1501), width, length)
    dy = make_rng(1502).standard_normal((width, length))
    _, saveds = hyena.layout_forward_saved(x, stack)
    dx, lg = hyena.layout_backward(stack, saveds, dy)
    for i, cfg in enumerate(layers):
        c.update(cfg_arrays(f"lay{i}", cfg))
        c.update(grads_arrays(f"lg{i}", lg[i]))
    c["lay.x"], c["lay.dy"], c["lay.dx"] = x.data, dy, dx
    # sharded a2a backward
    n = 0
    for n_ranks, d, dg, length, lh, layout in ((2, 4, 1, 32, 3, "sequential"), (4, 8, 2, 64, 5, "zigzag"),
                                               (4, 8, 1, 64, 5, "sequential")):
        rng = make_rng(1600 + n)
        groups = random_explicit_groups(rng, d, dg, lh)
        x = random_seq(rng, d, length)
        w = rng.standard_normal((d, length))
        grp = cpsim.SimGroup(n_ranks)
        _, asaved = cpsim.a2a_conv_saved(cpsim.shard(x, n_ranks, layout), groups, grp)
        dxs = cpsim.a2a_conv_backward(asaved, cpsim.shard(SeqTensor(w), n_ranks, layout), grp)
        c[f"ab{n}.args"] = np.array([str(n_ranks), str(d), str(dg), str(length), str(lh), layout])
        c[f"ab{n}.x"], c[f"ab{n}.dy"], c[f"ab{n}.taps"] = x.data, w, groups.materialized()
        c[f"ab{n}.dx"] = cpsim.gather(dxs).data
        c[f"ab{n}.elements"] = grp.total_elements("a2a_conv")
        c[f"ab{n}.messages"] = grp.total_messages("a2a_conv")
        n += 1
    c["n_ab"] = n
    save("backward", c)


if __name__ == "__main__":
    gen_direct()
    gen_blockconv()
    gen_fft()
    gen_filters()
    gen_hyena()
    gen_layout()
    gen_cpsim()
    gen_dfft()
    gen_builders()
    gen_backward()
