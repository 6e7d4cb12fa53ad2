"""GPU parity of the backward API against the reference-generated golden vectors and the
oracle restatement (oracle/backward.py):

* reference API (fp64 on the device): causal_conv_{input,taps}_grad, two_stage_backward,
  hyena_backward (every variant / backend / dtype of the goldens, factored projections),
  layout_backward;
* the device operator backward (operator_backward) in fp32 and bf16 against the oracle.

Tolerances (rel_err, testing.py:57-62): fp64 1e-10, fp32 1e-5, bf16 2e-2 for the chained
bf16 backward (each stage rounds to bf16; the fp64 oracle runs on bf16-representable inputs)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2503_01868_b200 as hy
from oracle import backward as ob

from .helpers import grads_from_golden, load, oracle_cfg, product_cfg

pytestmark = pytest.mark.gpu

Z = load("backward")


def _cfg_with_factored(z, prefix):
    cfg = product_cfg(z, prefix)
    if f"{prefix}.w_v.left" in z:
        import dataclasses
        cfg = dataclasses.replace(cfg, w_v=(z[f"{prefix}.w_v.left"], z[f"{prefix}.w_v.right"]))
    return cfg


def _check(g, want, tol, tag):
    assert oracle.rel_err(g.dx, want["dx"]) < tol, (tag, "dx")
    for name in ("dw_q", "dw_k", "dw_v", "dw_out"):
        a, b = getattr(g, name), want[name]
        if isinstance(b, tuple):
            assert oracle.rel_err(a[0], b[0]) < tol and oracle.rel_err(a[1], b[1]) < tol, (tag, name)
        else:
            assert oracle.rel_err(a, b) < tol, (tag, name)
    for role, per_group in g.filters.items():
        for leaf, arr in want["filters"][role].items():
            got = np.stack([d[leaf] for d in per_group])
            assert oracle.rel_err(got, arr) < tol, (tag, role, leaf)


def test_conv_adjoints_api_golden():
    for n in range(int(Z["n_cg"])):
        p = f"cg{n}"
        gs = int(Z[f"{p}.gs"])
        taps = Z[f"{p}.taps"]
        groups = hy.GroupSpec(taps.shape[0] * gs, gs, tuple(hy.ExplicitFilter(t) for t in taps))
        assert oracle.rel_err(hy.causal_conv_input_grad(Z[f"{p}.dy"], groups.taps_per_channel()),
                              Z[f"{p}.dx"]) < 1e-10
        assert oracle.rel_err(hy.causal_conv_taps_grad(Z[f"{p}.dy"], Z[f"{p}.x"], groups), Z[f"{p}.dtaps"]) < 1e-10


def test_two_stage_backward_api_golden():
    _, saved = hy.two_stage_forward_saved(hy.SeqTensor([[1.0, 2.0, 3.0, 4.0]]), hy.uniform_groups(1, [1.0, 1.0]), 2)
    g = hy.two_stage_backward(saved, np.ones((1, 4)))
    assert np.allclose(g.dtaps, [[10.0, 6.0]], atol=1e-12) and np.allclose(g.dv, [[2.0, 2.0, 2.0, 1.0]], atol=1e-12)
    for n in range(int(Z["n_tb"])):
        p = f"tb{n}"
        gs = int(Z[f"{p}.gs"])
        taps = Z[f"{p}.taps"]
        groups = hy.GroupSpec(taps.shape[0] * gs, gs, tuple(hy.ExplicitFilter(t) for t in taps))
        v = Z[f"{p}.v"]
        dt = "f32" if v.dtype == np.float32 else "f64"
        gated = f"{p}.q" in Z
        _, saved = hy.two_stage_forward_saved(
            hy.SeqTensor(v, dt), groups, int(Z[f"{p}.lb"]),
            q=hy.SeqTensor(Z[f"{p}.q"], dt) if gated else None, k=hy.SeqTensor(Z[f"{p}.k"], dt) if gated else None)
        g = hy.two_stage_backward(saved, Z[f"{p}.dy"])
        assert oracle.rel_err(g.dv, Z[f"{p}.dv"]) < 1e-10, p
        assert oracle.rel_err(g.dtaps, Z[f"{p}.dtaps"]) < 1e-10, p
        if gated:
            assert oracle.rel_err(g.dq, Z[f"{p}.dq"]) < 1e-10 and oracle.rel_err(g.dk, Z[f"{p}.dk"]) < 1e-10, p
    with pytest.raises(ValueError):
        hy.two_stage_backward(object(), np.ones((1, 4)))


@pytest.mark.parametrize("n", range(10))
def test_hyena_backward_api_golden(n):
    p = f"hb{n}"
    args = Z[f"{p}.args"]
    cfg = _cfg_with_factored(Z, f"{p}.cfg")
    x = Z[f"{p}.x"]
    dt = "f32" if x.dtype == np.float32 else "f64"
    y, saved = hy.hyena_forward_saved(hy.SeqTensor(x, dt), cfg)
    tol = 1e-10 if dt == "f64" else 1e-5
    assert oracle.rel_err(y.data, Z[f"{p}.y"]) < max(tol, 1e-6), (p, args)
    g = hy.hyena_backward(saved, Z[f"{p}.dy"])
    _check(g, grads_from_golden(Z, f"{p}.g"), tol, (p, tuple(args)))
    # parameter traversal (hyena.py:291-319) covers every leaf with a gradient of its shape
    for path, value in hy.iter_params(cfg):
        assert np.shape(hy.grad_for_path(g, path)) == np.shape(value), path


def test_layout_backward_api_golden():
    layers = tuple(_cfg_with_factored(Z, f"lay{i}") for i in range(3))
    stack = hy.OperatorStack(layers, residual=True)
    _, saveds = hy.layout_forward_saved(hy.SeqTensor(Z["lay.x"]), stack)
    dx, lg = hy.layout_backward(stack, saveds, Z["lay.dy"])
    assert oracle.rel_err(dx, Z["lay.dx"]) < 1e-10
    for i, g in enumerate(lg):
        _check(g, grads_from_golden(Z, f"lg{i}"), 1e-10, f"layer{i}")


# ---------------------------------------------------------------- device operator backward


def _bf16(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).double().numpy()


def _rounded_cfg(cfg, rnd):
    import dataclasses
    rc = {n: rnd(getattr(cfg, n)) for n in ("w_q", "w_k", "w_v", "w_out")}

    def rb(g):
        fs = []
        for f in g.filters:
            if isinstance(f, hy.ExplicitFilter):
                fs.append(hy.ExplicitFilter(rnd(f.taps)))
            elif isinstance(f, hy.RegularizedFilter):
                fs.append(hy.RegularizedFilter(rnd(f.taps_hat), f.decay_rate, f.base))
            else:
                fs.append(hy.ImplicitFilter(rnd(f.residues), rnd(f.poles), f.length))
        return hy.GroupSpec(g.channels, g.group_size, tuple(fs))

    return dataclasses.replace(cfg, **rc, **{n: rb(getattr(cfg, n)) for n in ("q_feat", "k_feat", "v_feat", "inner")})


def _oracle_cfg_of(cfg):
    def bank(g):
        fs = []
        for f in g.filters:
            if isinstance(f, hy.ExplicitFilter):
                fs.append(("explicit", f.taps))
            elif isinstance(f, hy.RegularizedFilter):
                fs.append(("regularized", f.taps_hat, f.decay_rate, f.base))
            else:
                fs.append(("implicit", f.residues, f.poles, f.length))
        return {"channels": g.channels, "group_size": g.group_size, "filters": fs}
    return {"variant": cfg.variant, "width": cfg.width, "block_size": cfg.block_size, "backend": "direct",
            **{n: getattr(cfg, n) for n in ("w_q", "w_k", "w_v", "w_out")},
            **{n: bank(getattr(cfg, n)) for n in ("q_feat", "k_feat", "v_feat", "inner")}}


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("variant,D,L,gs", [("SE", 16, 1024, 1), ("MR", 16, 2048, 2), ("LI", 16, 4096, 1),
                                             ("MR300", 16, 2048, 1)])
def test_operator_backward_vs_oracle(dtype, variant, D, L, gs):
    B = 2
    rng = hy.make_rng(77)
    lh = 300 if variant == "MR300" else 128  # MR300: bf16 forward / du on the K-block tcgen05 conv
    variant = "MR" if variant == "MR300" else variant
    kw = {"seq_len": L} if variant == "LI" else {"inner_len": lh if variant == "MR" else None}
    cfg = hy.make_hyena_config(variant, D, rng, group_size=gs, block_size=128 if variant == "MR" else 16, **kw)
    rnd = _bf16 if dtype == "bf16" else (lambda a: np.asarray(a, dtype=np.float32).astype(np.float64))
    cfg = _rounded_cfg(cfg, rnd)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = rnd(np.random.default_rng(1).standard_normal((B, D, L)))
    dy = rnd(np.random.default_rng(2).standard_normal((B, D, L)))
    op = hy.HyenaOperator(cfg, tdt)
    dx, g = hy.operator_backward(op, torch.from_numpy(x).to("cuda", tdt), torch.from_numpy(dy).to("cuda", tdt))
    ocfg = _oracle_cfg_of(cfg)
    want = None
    for b in range(B):
        _, saved = ob.hyena_forward_saved(x[b], ocfg)
        gb = ob.hyena_backward(saved, dy[b])
        if want is None:
            want = gb
            want["dx"] = [gb["dx"]]
        else:
            want["dx"].append(gb["dx"])
            for name in ("dw_q", "dw_k", "dw_v", "dw_out"):
                want[name] = want[name] + gb[name]
            for role in gb["filters"]:
                for gi, d in enumerate(gb["filters"][role]):
                    for leaf in d:
                        want["filters"][role][gi][leaf] = want["filters"][role][gi][leaf] + d[leaf]
    tol = 1e-5 if dtype == "f32" else 2e-2
    tol_p = 1e-4 if dtype == "f32" else 2e-2  # long fp32 reductions (B*L terms) for parameter grads
    assert oracle.rel_err(dx.double().cpu().numpy(), np.stack(want["dx"])) < tol
    wq = g.w_qkv_t.double().cpu().numpy()
    for i, name in enumerate(("dw_q", "dw_k", "dw_v")):
        assert oracle.rel_err(wq[i * D:(i + 1) * D].T, want[name]) < tol_p, name
    assert oracle.rel_err(g.w_out_t.double().cpu().numpy().T, want["dw_out"]) < tol_p
    ft = g.feat_taps.double().cpu().numpy()
    for i, role in enumerate(("q_feat", "k_feat", "v_feat")):
        fgs = getattr(cfg, role).group_size  # device taps are per channel: sum over each group
        got = ft[i, :, :cfg.q_feat.filter_len].reshape(D // fgs, fgs, -1).sum(1)
        exp = np.stack([d["taps"] for d in want["filters"][role]])
        assert oracle.rel_err(got, exp) < tol_p, role
    for leaf, arr in g.inner.items():
        exp = np.stack([d[leaf] for d in want["filters"]["inner"]])
        assert oracle.rel_err(arr.double().cpu().numpy(), exp) < tol_p, ("inner", leaf)
