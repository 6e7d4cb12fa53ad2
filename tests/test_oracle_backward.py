"""The oracle's backward restatement (oracle/backward.py) against golden vectors produced by
the reference's own backward (tests/golden/make_golden.py gen_backward). CPU only."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from oracle import backward as ob

from .helpers import grads_from_golden, load, oracle_cfg, stack_filter_grads

Z = load("backward")
TOL = 1e-10


def _rel(a, b):
    return oracle.rel_err(a, b)


def test_conv_adjoints_golden():
    for n in range(int(Z["n_cg"])):
        p = f"cg{n}"
        gs = int(Z[f"{p}.gs"])
        taps = Z[f"{p}.taps"]
        bank = oracle.explicit_bank(taps.shape[0] * gs, gs, taps)
        assert _rel(ob.causal_conv_input_grad(Z[f"{p}.dy"], np.repeat(taps, gs, axis=0)), Z[f"{p}.dx"]) < TOL
        assert _rel(ob.causal_conv_taps_grad(Z[f"{p}.dy"], Z[f"{p}.x"], bank), Z[f"{p}.dtaps"]) < TOL


def test_two_stage_backward_hand_example():
    """pkg/tests/test_blockconv.py:154-160: h=[1,1], v=[1,2,3,4], dy=1 -> dtaps [10, 6], dv [2,2,2,1]."""
    _, saved = ob.two_stage_forward_saved(np.array([[1.0, 2.0, 3.0, 4.0]]), oracle.uniform_bank(1, [1.0, 1.0]), 2)
    g = ob.two_stage_backward(saved, np.ones((1, 4)))
    assert np.array_equal(g["dtaps"], [[10.0, 6.0]]) and np.array_equal(Z["hand.dtaps"], [[10.0, 6.0]])
    assert np.array_equal(g["dv"], [[2.0, 2.0, 2.0, 1.0]]) and np.array_equal(g["dv"], Z["hand.dv"])


def test_two_stage_backward_golden():
    for n in range(int(Z["n_tb"])):
        p = f"tb{n}"
        gs = int(Z[f"{p}.gs"])
        taps = Z[f"{p}.taps"]
        bank = oracle.explicit_bank(taps.shape[0] * gs, gs, taps)
        gated = f"{p}.q" in Z
        _, saved = ob.two_stage_forward_saved(Z[f"{p}.v"], bank, int(Z[f"{p}.lb"]),
                                              q=Z[f"{p}.q"] if gated else None, k=Z[f"{p}.k"] if gated else None)
        g = ob.two_stage_backward(saved, Z[f"{p}.dy"])
        assert _rel(g["dv"], Z[f"{p}.dv"]) < TOL, p
        assert _rel(g["dtaps"], Z[f"{p}.dtaps"]) < TOL, p
        if gated:
            assert _rel(g["dq"], Z[f"{p}.dq"]) < TOL, p
            assert _rel(g["dk"], Z[f"{p}.dk"]) < TOL, p


def _check_grads(g: dict, want: dict, tag: str):
    assert _rel(g["dx"], want["dx"]) < TOL, (tag, "dx")
    for name in ("dw_q", "dw_k", "dw_v", "dw_out"):
        a, b = g[name], want[name]
        if isinstance(b, tuple):
            assert _rel(a[0], b[0]) < TOL and _rel(a[1], b[1]) < TOL, (tag, name)
        else:
            assert _rel(a, b) < TOL, (tag, name)
    for role, per_group in g["filters"].items():
        got = stack_filter_grads(per_group)
        for leaf, arr in want["filters"][role].items():
            assert _rel(got[leaf], arr) < TOL, (tag, role, leaf)


@pytest.mark.parametrize("n", range(10))
def test_hyena_backward_golden(n):
    p = f"hb{n}"
    if n >= int(Z["n_hb"]):
        pytest.skip("no such case")
    cfg = oracle_cfg(Z, f"{p}.cfg")
    y, saved = ob.hyena_forward_saved(Z[f"{p}.x"], cfg)
    assert _rel(y, Z[f"{p}.y"]) < 1e-6
    _check_grads(ob.hyena_backward(saved, Z[f"{p}.dy"]), grads_from_golden(Z, f"{p}.g"), p)


def test_layout_backward_golden():
    layers = [oracle_cfg(Z, f"lay{i}") for i in range(3)]
    _, saveds = ob.layout_forward_saved(Z["lay.x"], layers, residual=True)
    dx, grads = ob.layout_backward(layers, saveds, Z["lay.dy"], residual=True)
    assert _rel(dx, Z["lay.dx"]) < TOL
    for i, g in enumerate(grads):
        _check_grads(g, grads_from_golden(Z, f"lg{i}"), f"layer{i}")


def test_a2a_backward_golden_is_the_input_adjoint():
    """cpsim.py:440-446: the sharded backward equals the unsharded conv input adjoint."""
    for n in range(int(Z["n_ab"])):
        p = f"ab{n}"
        dg = int(Z[f"{p}.args"][2])
        taps = Z[f"{p}.taps"]
        assert _rel(ob.causal_conv_input_grad(Z[f"{p}.dy"], np.repeat(taps, dg, axis=0)), Z[f"{p}.dx"]) < TOL
