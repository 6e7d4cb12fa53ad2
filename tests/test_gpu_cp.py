"""GPU checks of the context-parallel path.

* single GPU: the fused mixer with a projection history equals the second half of a
  full-sequence run (the property the CP operator relies on);
* >= 2 GPUs (skipped otherwise): HyenaCP over NCCL equals the single-GPU operator.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import ops

pytestmark = pytest.mark.gpu


def test_mixer_history_equals_split():
    g = torch.Generator(device="cuda").manual_seed(3)
    B, C, L = 2, 16, 8192
    proj = torch.randn((B, 3 * C, L), device="cuda", dtype=torch.bfloat16, generator=g)
    feat = torch.randn((3, C, 7), device="cuda", generator=g) / 3
    taps = torch.randn((C, 128), device="cuda", generator=g) / 11
    decay = torch.linspace(0.01, 2.0, C, device="cuda")
    full = ops.hyena_mixer(proj, feat, taps, 1, decay=decay)
    for cut in (4096, 2048, 512):
        hist = proj[..., cut - 144:cut].contiguous()
        second = ops.hyena_mixer(proj[..., cut:].contiguous(), feat, taps, 1, decay=decay, hist=hist)
        assert torch.equal(second, full[..., cut:]), cut


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cp_worker(rank, world, port, variant, q, p2p="1", batch=1):
    import torch.distributed as dist
    os.environ["HY_CP_P2P"] = p2p
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        D, L = 64, 8192 * world
        kw = {"inner_len": 128, "block_size": 128} if variant == "MR" else {}
        cfg = hy.make_hyena_config(variant, D, hy.make_rng(0), seq_len=L, **kw)
        gen = torch.Generator(device="cuda").manual_seed(7)
        x = torch.randn((batch, D, L), device="cuda", dtype=torch.bfloat16, generator=gen)
        m = L // world
        cpop = hy.cp.HyenaCP(cfg, torch.bfloat16)
        for _ in range(3):  # repeated steps exercise the slot flow control of the peer transfers
            y_local = cpop.forward(x[..., rank * m:(rank + 1) * m].contiguous())
        if rank == 0:
            y_ref = hy.HyenaOperator(cfg, torch.bfloat16).forward(x)
        parts = [torch.empty_like(y_local) for _ in range(world)]
        dist.all_gather(parts, y_local)
        if rank == 0:
            y = torch.cat(parts, dim=-1).float()
            err = float((y - y_ref.float()).abs().max() / max(1.0, float(y_ref.float().abs().max())))
            q.put(err)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("p2p", ["1", "0"], ids=["peer", "nccl"])
@pytest.mark.parametrize("variant", ["MR", "SE", "LI"])
def test_hyena_cp_matches_single_gpu(variant, p2p):
    """HyenaCP's halo / all-to-all over copy-engine peer transfers (default) and over NCCL."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cp_worker, args=(r, world, port, variant, q, p2p)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert err < 2e-2, err


def _a2a_bwd_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from oracle import backward as ob
        D, L, lh = 16, 4096, 9
        rng = np.random.default_rng(5)
        taps = rng.standard_normal((D // 2, lh)) / 3
        groups = hy.GroupSpec(D, 2, tuple(hy.ExplicitFilter(t) for t in taps))
        x = rng.standard_normal((D, L))
        dy = rng.standard_normal((D, L))
        grp = hy.cp.CPGroup()
        res = {}
        for layout in ("sequential", "zigzag"):
            xs = hy.cp.shard(hy.SeqTensor(x), world, layout)
            dys = hy.cp.shard(hy.SeqTensor(dy), world, layout)
            _, saved = hy.cp.a2a_conv_saved(torch.from_numpy(xs.shards[rank].copy()).cuda(), groups, grp, layout)
            dx = hy.cp.a2a_conv_backward(saved, torch.from_numpy(dys.shards[rank].copy()).cuda(), grp)
            parts = [torch.empty_like(dx) for _ in range(world)]
            dist.all_gather(parts, dx)
            if rank == 0:
                got = hy.cp.gather(hy.cp.ShardedSeq([p.cpu().numpy() for p in parts], layout)).data
                want = ob.causal_conv_input_grad(dy, np.repeat(taps, 2, axis=0))
                res[layout] = float(np.abs(got - want).max() / max(1.0, np.abs(want).max()))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_hyena_cp_li_batched():
    """LI CP layer with B = 2: the software pipeline's peer slots cycle through both batch
    elements of every segment (flow control across segments)."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cp_worker, args=(r, world, port, "LI", q, "1", 2)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert err < 2e-2, err


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_a2a_backward_nccl_matches_oracle():
    """a2a_conv_backward (cpsim.py:440-446) over NCCL, fp64 slab adjoint on the device, both
    layouts, against the oracle's unsharded input adjoint (core.py:245-252)."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_bwd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for layout, err in res.items():
        assert err < 1e-12, (layout, err)


def _layout_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        D, L = 64, 8192 * world
        rng = hy.make_rng(4)
        layers = (hy.make_hyena_config("SE", D, rng, seq_len=L),
                  hy.make_hyena_config("MR", D, rng, inner_len=128, block_size=128),
                  hy.make_hyena_config("LI", D, rng, seq_len=L),
                  hy.make_hyena_config("MR", D, rng, inner_len=128, block_size=128))
        stack = hy.build_layout(hy.LayoutSpec(("SE", "MR", "LI", "MR"), 1, layers), residual=True)
        gen = torch.Generator(device="cuda").manual_seed(9)
        x = torch.randn((1, D, L), device="cuda", dtype=torch.bfloat16, generator=gen)
        m = L // world
        lcp = hy.LayoutCP(stack, torch.bfloat16)
        for _ in range(2):
            y_local = lcp.forward(x[..., rank * m:(rank + 1) * m].contiguous())
        parts = [torch.empty_like(y_local) for _ in range(world)]
        dist.all_gather(parts, y_local)
        if rank == 0:
            y_ref = hy.layout_forward_device(x, stack).float()
            y = torch.cat(parts, dim=-1).float()
            q.put(float((y - y_ref).abs().max() / max(1.0, float(y_ref.abs().max()))))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_layout_cp_matches_single_gpu():
    """SE-MR-LI-MR residual stack sharded once across ranks (LayoutCP) equals the single-GPU
    layout forward; the layers share the group's peer buffers."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_layout_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert err < 2e-2, err


def _dfft_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import oracle
        rng = np.random.default_rng(21)
        C, L, lh = 4, 3000, 700
        x = rng.standard_normal((C, L))
        taps = rng.standard_normal((C, lh)) / np.sqrt(lh)
        y = hy.cp.p2p_fft_causal_wrapper(hy.SeqTensor(x), taps, hy.cp.CPGroup())
        if rank == 0:
            want = oracle.direct_causal_conv(x, {"channels": C, "group_size": 1,
                                                 "filters": [("explicit", t) for t in taps]})
            q.put(float(np.abs(y.data - want).max() / max(1.0, np.abs(want).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_p2p_fft_causal_nccl_matches_oracle():
    """Distributed FFT conv (cpsim.py:634-659) over NCCL on the devices, float64 (cuFFT local
    transforms), against the oracle's direct causal conv."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dfft_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert err < 1e-10, err
