"""Context-parallel schemes over torch.distributed on CPU (gloo, world size 2 and 4),
checked against the reference's own simulator outputs (tests/golden/cpsim.npz).

The local convolutions are injected (the oracle's direct conv) so these tests exercise
the host-side logic — sharding, halo exchange, all-to-all permutation, accounting —
without a GPU. The GPU path uses the same functions with the sm_100a kernels.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from .helpers import explicit_bank_from_taps, load, product_groups_from_taps


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    import oracle
    from paper_2503_01868_b200 import cp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scheme, n_ranks, layout, n_pipe = case["scheme"], case["n_ranks"], case["layout"], case["n_pipe"]
        gs = case["gs"]
        taps = case["taps"]
        groups = product_groups_from_taps(taps, gs)
        bank = explicit_bank_from_taps(taps, gs)
        xs = cp.shard(__import__("paper_2503_01868_b200").SeqTensor(case["x"]), n_ranks, layout)
        local = torch.from_numpy(xs.shards[rank].copy())
        grp = cp.CPGroup()

        def conv(x):
            return torch.from_numpy(np.asarray(oracle.direct_causal_conv(x.numpy(), bank), dtype=np.float64))

        def correct(halo, y):
            H = halo.shape[-1]
            ov = np.concatenate([halo.numpy(), np.zeros_like(halo.numpy())], axis=1)
            y = y.clone()
            y[:, :H] += torch.from_numpy(oracle.direct_causal_conv(ov, bank)[:, H:])
            return y

        def conv_slab(natural, slab_groups):
            b = explicit_bank_from_taps(slab_groups.materialized(), slab_groups.group_size)
            return torch.from_numpy(oracle.direct_causal_conv(natural.numpy(), b))

        if scheme == "p2p":
            y = cp.p2p_conv(local, groups, grp, layout, conv=conv)
        elif scheme == "p2p_ov":
            y = cp.p2p_conv_overlapped(local, groups, grp, layout, conv=conv, correct=correct)
        elif scheme == "a2a":
            y = cp.a2a_conv(local, groups, grp, layout, conv_slab=conv_slab)
        else:
            y = cp.a2a_conv_pipelined(local, groups, grp, n_pipe, layout, conv_slab=conv_slab)
        q.put((rank, y.numpy(), grp.total_elements(case["name"]), grp.total_messages(case["name"]),
               grp.scheme_rounds.get(case["name"], 0), [grp.filter_elements[r] for r in range(n_ranks)]))
    finally:
        dist.destroy_process_group()


def _cases():
    z = load("cpsim")
    out = []
    for i in range(int(z["n_cp"])):
        scheme, n_ranks, d, dg, length, lh, n_pipe, layout, name = [str(a) for a in z[f"cp{i}.args"]]
        out.append(dict(idx=i, scheme=scheme, n_ranks=int(n_ranks), gs=int(dg), n_pipe=int(n_pipe), layout=layout,
                        name=name, taps=z[f"cp{i}.taps"], x=z[f"cp{i}.x"],
                        shards=[z[f"cp{i}.shard{r}"] for r in range(int(n_ranks))],
                        elements=int(z[f"cp{i}.elements"]), messages=int(z[f"cp{i}.messages"]),
                        rounds=int(z[f"cp{i}.rounds"]), filter_elements=list(z[f"cp{i}.filter_elements"])))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['scheme']}-{c['n_ranks']}r-{c['layout']}-{c['idx']}")
def test_cp_scheme_matches_reference_simulator(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, case["n_ranks"], port, case, q)) for r in range(case["n_ranks"])]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, y, el, msg, rounds, fe = q.get(timeout=180)
        res[rank] = (y, el, msg, rounds, fe)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(case["n_ranks"]):
        y, el, msg, rounds, fe = res[r]
        assert np.max(np.abs(y - case["shards"][r])) < 1e-12, r
        assert el == case["elements"] and msg == case["messages"], (el, msg)
        assert rounds == case["rounds"]
        assert fe == case["filter_elements"]


def test_shard_gather_roundtrip_and_layouts():
    from paper_2503_01868_b200 import SeqTensor, cp
    x = SeqTensor(np.arange(16.0)[None, :])
    zz = cp.shard(x, 4, "zigzag")
    assert list(zz.shards[0][0]) == [0.0, 1.0, 14.0, 15.0]
    assert list(zz.shards[3][0]) == [6.0, 7.0, 8.0, 9.0]
    assert np.array_equal(cp.gather(zz).data, x.data)
    seq = cp.shard(SeqTensor(np.arange(8.0)[None, :]), 4)
    assert [list(s[0]) for s in seq.shards] == [[0.0, 1.0], [2.0, 3.0], [4.0, 5.0], [6.0, 7.0]]
    with pytest.raises(ValueError):
        cp.shard(SeqTensor(np.zeros((2, 30))), 4)
    with pytest.raises(ValueError):
        cp.shard(SeqTensor(np.zeros((2, 12))), 4, "zigzag")


def _bwd_worker(rank, world, port, case, q):
    from oracle import backward as ob
    from paper_2503_01868_b200 import SeqTensor, cp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gs, layout = case["gs"], case["layout"]
        groups = product_groups_from_taps(case["taps"], gs)
        grp = cp.CPGroup()
        xs = cp.shard(SeqTensor(case["x"]), world, layout)
        dys = cp.shard(SeqTensor(case["dy"]), world, layout)

        def conv_slab(natural, slab_groups):
            b = explicit_bank_from_taps(slab_groups.materialized(), slab_groups.group_size)
            return torch.from_numpy(__import__("oracle").direct_causal_conv(natural.numpy(), b))

        def slab_bwd(natural, slab_groups):
            tpc = np.repeat(slab_groups.materialized(), slab_groups.group_size, axis=0)
            return torch.from_numpy(ob.causal_conv_input_grad(natural.numpy(), tpc))

        _, saved = cp.a2a_conv_saved(torch.from_numpy(xs.shards[rank].copy()), groups, grp, layout,
                                     conv_slab=conv_slab)
        fwd_el = grp.total_elements("a2a_conv")
        dx = cp.a2a_conv_backward(saved, torch.from_numpy(dys.shards[rank].copy()), grp, conv_slab=slab_bwd)
        q.put((rank, dx.numpy(), grp.total_elements("a2a_conv") - fwd_el, grp.total_elements("a2a_conv"),
               grp.total_messages("a2a_conv")))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("idx", range(3))
def test_a2a_backward_matches_reference(idx):
    """a2a_conv_backward (cpsim.py:440-446) on gloo vs the reference's sharded backward:
    gathered dx, and the accounting (forward + backward both counted under a2a_conv)."""
    from paper_2503_01868_b200 import SeqTensor, cp
    z = load("backward")
    n_ranks, d, dg, length, lh, layout = [str(a) for a in z[f"ab{idx}.args"]]
    n_ranks = int(n_ranks)
    case = dict(gs=int(dg), layout=layout, taps=z[f"ab{idx}.taps"], x=z[f"ab{idx}.x"], dy=z[f"ab{idx}.dy"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bwd_worker, args=(r, n_ranks, port, case, q)) for r in range(n_ranks)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, dx, bwd_el, tot_el, tot_msg = q.get(timeout=180)
        res[rank] = (dx, bwd_el, tot_el, tot_msg)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = [res[r][0] for r in range(n_ranks)]
    got = cp.gather(cp.ShardedSeq(shards, layout)).data
    assert np.max(np.abs(got - z[f"ab{idx}.dx"])) < 1e-12
    assert res[0][2] == int(z[f"ab{idx}.elements"]) and res[0][3] == int(z[f"ab{idx}.messages"])
    assert res[0][1] * 2 == res[0][2]  # the backward moves as much as the forward


def _dfft_worker(rank, world, port, q):
    from paper_2503_01868_b200 import SeqTensor, cp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = load("dfft")
        out = {}
        if f"own{world}.x" in z:  # bin ownership of the forward transform
            grp = cp.CPGroup()
            x = z[f"own{world}.x"]
            m = x.shape[-1] // world
            spec = cp.p2p_fft_forward(torch.from_numpy(x[:, rank * m:(rank + 1) * m].copy()), grp)
            out["own"] = float(np.max(np.abs(spec.numpy() - z[f"own{world}.spec{rank}"])))
        grp = cp.CPGroup()
        x, h = z[f"conv{world}.x"], z[f"conv{world}.h"]
        m = x.shape[-1] // world
        lx = torch.from_numpy(x[:, rank * m:(rank + 1) * m].copy())
        lh = torch.from_numpy(h[:, rank * m:(rank + 1) * m].copy())
        y = cp.p2p_fft_conv(lx, lh, grp)
        out["conv"] = float(np.max(np.abs(y.numpy() - z[f"conv{world}.y"][:, rank * m:(rank + 1) * m])))
        out["acct"] = (grp.total_elements("p2p_fft_conv"), grp.total_messages("p2p_fft_conv"),
                       grp.scheme_rounds.get("p2p_fft_conv", 0), max(grp.max_resident.values()))
        out["want_acct"] = (int(z[f"conv{world}.elements"]), int(z[f"conv{world}.messages"]),
                            int(z[f"conv{world}.rounds"]), int(z[f"conv{world}.max_resident"]))
        for case, n in (("causal", 4), ("trunc", 2)):
            if n == world:
                yc = cp.p2p_fft_causal_wrapper(SeqTensor(z[f"{case}.x"]), z[f"{case}.taps"], cp.CPGroup())
                out[case] = float(np.max(np.abs(yc.data - z[f"{case}.y"])))
        if world == 2:  # the reference's argument checks (test_cpsim.py:391-402)
            for bad in (lambda: cp.p2p_fft_forward(torch.zeros((1, 12), dtype=torch.float64), cp.CPGroup()),
                        lambda: cp.p2p_fft_conv(torch.zeros((2, 16), dtype=torch.float64),
                                                torch.zeros((1, 16), dtype=torch.float64), cp.CPGroup())):
                try:
                    bad()
                    out["raises"] = False
                except ValueError:
                    out.setdefault("raises", True)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p2p_fft_matches_reference_simulator(world):
    """Distributed FFT over gloo (cpsim.py:537-659) against the reference simulator's outputs:
    bit-reversed bin ownership, circular conv, accounting, causal wrapper, argument checks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dfft_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, out in res.items():
        assert out.get("own", 0.0) < 1e-10, (r, out)
        assert out["conv"] < 1e-10, (r, out)
        assert out["acct"] == out["want_acct"], (r, out)
        assert out.get("causal", 0.0) < 1e-10 and out.get("trunc", 0.0) < 1e-10, (r, out)
        assert out.get("raises", True), (r, out)


def _zigzag_worker(rank, world, port, q):
    import oracle
    from paper_2503_01868_b200 import SeqTensor, cp
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        C, L, lh = 3, 32 * world, 5
        taps = rng.standard_normal((C, lh))
        x = rng.standard_normal((C, L))
        bank = explicit_bank_from_taps(taps, 1)
        local = cp.shard(SeqTensor(x), world, "zigzag").shards[rank]
        h, H = local.shape[1] // 2, lh - 1
        grp = cp.CPGroup()
        a, b = torch.from_numpy(local[:, :h].copy()), torch.from_numpy(local[:, h:].copy())
        hist = cp._zigzag_history(a[None, :, h - H:].contiguous(), b[None, :, h - H:].contiguous(), grp, "zz")
        outs = []
        for half, hh in ((a, hist[0]), (b, hist[1])):
            ext = np.concatenate([hh.numpy(), half.numpy()], axis=1)
            outs.append(oracle.direct_causal_conv(ext, bank)[:, H:])
        q.put((rank, np.concatenate(outs, axis=1), grp.total_messages("zz"), grp.scheme_rounds.get("zz", 0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_zigzag_history_host_logic(world):
    """The zigzag layout's two causal halos (cp._zigzag_history): each half, convolved after
    its history, reproduces its chunk of the unsharded conv; 2 (N - 1) messages, one round."""
    import oracle
    from paper_2503_01868_b200 import SeqTensor, cp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zigzag_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    C, L, lh = 3, 32 * world, 5
    taps = rng.standard_normal((C, lh))
    x = rng.standard_normal((C, L))
    want = oracle.direct_causal_conv(x, explicit_bank_from_taps(taps, 1))
    got = cp.gather(cp.ShardedSeq(tuple(r[1] for r in res), "zigzag")).data
    assert np.max(np.abs(got - want)) < 1e-12
    assert all(r[2] == 2 * (world - 1) and r[3] == 1 for r in res)
