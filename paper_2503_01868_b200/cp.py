"""Context-parallel convolution over torch.distributed (one process per GPU, NCCL).

Restates the reference's simulated schemes (/root/reference/pkg/src/convhybrid/cpsim.py)
as real collectives. Every rank holds one time shard `(C, L/N)` (or `(B, C, L/N)`) of
the sequence; the functions below take the rank's local tensor and return its local
output, and tally the same accounting as the reference's SimGroup (cpsim.py:69-131):

  p2p_conv             halo of lh-1 steps from rank r to r+1, conv on [halo | local]
                       (cpsim.py:460-495)
  p2p_conv_overlapped  local conv on zero history launched before the halo is consumed,
                       then the correction conv of the halo (cpsim.py:498-534)
  a2a_conv             two all_to_all_single rounds swap time shards <-> channel slabs,
                       conv over the full sequence on the slab (cpsim.py:325-447)
  a2a_conv_pipelined   the same in n_pipe channel segments (cpsim.py:449-454)
  p2p_fft_conv         distributed FFT: log2(N) cross-rank DiF stages (one partner
                       exchange each), local FFT, bit-reversed bin ownership, spectrum
                       product, inverse (cpsim.py:540-659)

`HyenaCP` composes them into the context-parallel Hyena operator:
projections and gates are token-local; SE/MR receive the last 144 steps of the
predecessor's projections and run the fused tcgen05 mixer with that history; LI swaps
u = k*v to channel slabs with all-to-all for the long convolution.
"""

from __future__ import annotations

import os

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import blas
from .core import GroupSpec, SeqTensor

LAYOUTS = ("sequential", "zigzag")


@dataclass
class CPGroup:
    """A torch.distributed process group plus the reference's accounting fields."""

    group: object = None  # torch.distributed ProcessGroup (None = default world group)
    scheme_elements: dict = field(default_factory=dict)
    scheme_messages: dict = field(default_factory=dict)
    scheme_rounds: dict = field(default_factory=dict)
    filter_elements: dict = field(default_factory=dict)
    message_log: list = field(default_factory=list)
    # symmetric peer buffers (p2p.PeerHalo / PeerAllToAll) shared by every CP layer on this
    # group, keyed by (kind, shape, dtype): a deep stack maps one set, not one per layer
    peers: dict = field(default_factory=dict, repr=False)
    max_resident: dict = field(default_factory=dict)  # rank -> max sequence samples held (dfft)

    def note_resident(self, rank: int, samples: int) -> None:
        self.max_resident[rank] = max(self.max_resident.get(rank, 0), samples)

    def peer(self, kind: str, shape, dtype, nslots: int = 2):
        """The shared peer exchanger, or None when the ranks cannot map each other's memory
        (then the callers use NCCL; every rank reaches the same answer)."""
        key = (kind, tuple(shape), dtype, nslots)
        if key not in self.peers:
            from . import p2p
            try:
                if kind == "halo":
                    self.peers[key] = p2p.PeerHalo(self.group, shape, dtype)
                else:  # the LI all-to-all: a scatter and a return exchanger
                    self.peers[key] = (p2p.PeerAllToAll(self.group, shape, dtype, nslots),
                                       p2p.PeerAllToAll(self.group, shape, dtype, nslots))
            except p2p.PeerUnavailable as e:
                import warnings
                warnings.warn(f"peer-memory transfers unavailable, using NCCL: {e}")
                self.peers[key] = None
        return self.peers[key]

    def close(self) -> None:
        """Release the group's peer exchangers (collective: every rank calls it)."""
        for key in sorted(self.peers, key=repr):
            ex = self.peers.pop(key)
            for e in (ex if isinstance(ex, tuple) else (ex,)):
                if e is not None:
                    e.close()

    def __post_init__(self):
        n = self.n_ranks
        if n < 1 or (n & (n - 1)) != 0:
            raise ValueError(f"rank count must be a power of two >= 1, got {n}")

    @property
    def n_ranks(self) -> int:
        return dist.get_world_size(self.group)

    @property
    def rank(self) -> int:
        return dist.get_rank(self.group)

    def _send(self, scheme: str, src: int, dst: int, elements: int) -> None:
        # every rank tallies every message of the scheme, so counters agree across ranks
        self.message_log.append((len(self.message_log) + 1, scheme, src, dst, int(elements)))
        self.scheme_elements[scheme] = self.scheme_elements.get(scheme, 0) + int(elements)
        self.scheme_messages[scheme] = self.scheme_messages.get(scheme, 0) + 1

    def count_rounds(self, scheme: str, n: int) -> None:
        self.scheme_rounds[scheme] = self.scheme_rounds.get(scheme, 0) + n

    def total_elements(self, scheme: str | None = None) -> int:
        return self.scheme_elements.get(scheme, 0) if scheme else sum(self.scheme_elements.values())

    def total_messages(self, scheme: str | None = None) -> int:
        return self.scheme_messages.get(scheme, 0) if scheme else sum(self.scheme_messages.values())


# ---------------------------------------------------------------- transport
# NCCL moves CUDA tensors itself. A gloo group (CPU-only collectives) that is handed CUDA
# tensors -- e.g. two ranks sharing one GPU, where NCCL refuses to run -- stages them
# through host memory; bf16 (no gloo type) travels as its bytes (no arithmetic on the way).


def _staged(grp: CPGroup, t: torch.Tensor) -> bool:
    return t.is_cuda and dist.get_backend(grp.group) != "nccl"


def _wire(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.uint8) if t.dtype == torch.bfloat16 else t


def _host_like(t: torch.Tensor) -> torch.Tensor:
    """An empty host buffer of t's wire shape and type."""
    return torch.empty(_wire(t).shape, dtype=_wire(t).dtype)


def _unwire(host: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    return host.view(like.dtype) if like.dtype == torch.bfloat16 else host


class _HostReq:
    """A gloo request on a host copy; wait() copies a received host buffer back."""

    def __init__(self, req, host, dst=None):
        self.req, self.host, self.dst = req, host, dst

    def wait(self):
        self.req.wait()
        if self.dst is not None:
            self.dst.copy_(_unwire(self.host, self.dst))
        return True


def _batch_p2p(grp: CPGroup, ops_) -> list:
    """ops_: [("send" | "recv", tensor, peer)] -> requests with wait()."""
    if not ops_:
        return []
    if not any(_staged(grp, t) for _, t, _ in ops_):
        return dist.batch_isend_irecv([dist.P2POp(dist.isend if k == "send" else dist.irecv, t, p, grp.group)
                                       for k, t, p in ops_])
    torch.cuda.synchronize()
    reqs = []
    for k, t, p in ops_:
        if k == "send":
            host = _wire(t.detach().contiguous()).cpu()
            reqs.append(_HostReq(dist.isend(host, p, group=grp.group), host))
        else:
            host = _host_like(t)
            reqs.append(_HostReq(dist.irecv(host, p, group=grp.group), host, t))
    return reqs


def _all_to_all(grp: CPGroup, out: torch.Tensor, inp: torch.Tensor) -> None:
    if not _staged(grp, inp):
        dist.all_to_all_single(out, inp, group=grp.group)
        return
    host = _host_like(out.contiguous())
    dist.all_to_all_single(host, _wire(inp.contiguous()).cpu(), group=grp.group)
    out.copy_(_unwire(host, out))


def _all_gather(grp: CPGroup, parts: list, t: torch.Tensor) -> None:
    if not _staged(grp, t):
        dist.all_gather(parts, t, group=grp.group)
        return
    hosts = [_host_like(p) for p in parts]
    dist.all_gather(hosts, _wire(t.contiguous()).cpu(), group=grp.group)
    for p, h in zip(parts, hosts):
        p.copy_(_unwire(h, p))


# ---------------------------------------------------------------- sharding (cpsim.py:244-319)


@dataclass(frozen=True)
class ShardedSeq:
    """Per-rank (d, l/n_ranks) slices of one sequence (host view, cpsim.py:247-279)."""

    shards: tuple
    layout: str = "sequential"

    def __post_init__(self):
        shards = tuple(np.asarray(s) for s in self.shards)
        if not shards:
            raise ValueError("need at least one shard")
        if any(s.shape != shards[0].shape for s in shards):
            raise ValueError("all shards must share one shape")
        if self.layout not in LAYOUTS:
            raise ValueError(f"layout must be one of {LAYOUTS}, got {self.layout!r}")
        object.__setattr__(self, "shards", shards)

    @property
    def n_ranks(self) -> int:
        return len(self.shards)

    @property
    def channels(self) -> int:
        return self.shards[0].shape[0]

    @property
    def shard_len(self) -> int:
        return self.shards[0].shape[1]

    @property
    def total_len(self) -> int:
        return self.shard_len * self.n_ranks


def layout_chunks(layout: str, n_ranks: int):
    """Chunk ids per rank in local time order; zigzag gives rank r chunks r and 2N-1-r."""
    if layout == "sequential":
        return [[r] for r in range(n_ranks)]
    return [[r, 2 * n_ranks - 1 - r] for r in range(n_ranks)]


def shard(x: SeqTensor, n_ranks: int, layout: str = "sequential") -> ShardedSeq:
    """(cpsim.py:289-301)."""
    if layout not in LAYOUTS:
        raise ValueError(f"layout must be one of {LAYOUTS}, got {layout!r}")
    divisor = n_ranks * (1 if layout == "sequential" else 2)
    if x.length % divisor != 0:
        raise ValueError(f"length {x.length} not divisible by {divisor} ({layout} layout over {n_ranks} ranks)")
    clen = x.length // divisor
    return ShardedSeq(tuple(np.concatenate([x.data[:, c * clen:(c + 1) * clen] for c in ids], axis=1)
                            for ids in layout_chunks(layout, n_ranks)), layout)


def gather(xs: ShardedSeq) -> SeqTensor:
    """(cpsim.py:304-312)."""
    ids = layout_chunks(xs.layout, xs.n_ranks)
    clen = xs.shard_len // len(ids[0])
    out = np.empty((xs.channels, xs.total_len), dtype=np.float64)
    for r, cs in enumerate(ids):
        for i, c in enumerate(cs):
            out[:, c * clen:(c + 1) * clen] = xs.shards[r][:, i * clen:(i + 1) * clen]
    return SeqTensor(out)


def natural_cols(layout: str, n_ranks: int, total_len: int) -> np.ndarray:
    """Assembled (rank-major) position i holds natural time column map[i] (cpsim.py:315-319)."""
    ids = [c for cs in layout_chunks(layout, n_ranks) for c in cs]
    clen = total_len // len(ids)
    return np.concatenate([np.arange(c * clen, (c + 1) * clen) for c in ids])


# ---------------------------------------------------------------- default (GPU) local kernels


def _gpu_conv(taps: torch.Tensor, gs: int):
    from . import ops

    def conv(x):
        return ops.long_conv(x.contiguous(), taps, gs) if taps.shape[-1] > 32 else ops.causal_conv(x.contiguous(), taps, gs)
    return conv


def _gpu_correct(taps: torch.Tensor, gs: int):
    from . import ops

    def correct(halo, y):
        ops.halo_correction(halo.contiguous(), y, taps, gs)
        return y
    return correct


def _taps_tensor(groups: GroupSpec, like: torch.Tensor) -> torch.Tensor:
    from .ops import tap_dtype
    dt = tap_dtype(like.dtype) if like.is_floating_point() else torch.float64
    return torch.from_numpy(groups.materialized()).to(like.device, dt)


# ---------------------------------------------------------------- p2p halo schemes


def _check_p2p(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, layout: str) -> int:
    if layout != "sequential":
        raise ValueError("point-to-point schemes need the sequential layout")
    if local.shape[-2] != groups.channels:
        raise ValueError(f"input has {local.shape[-2]} channels, grouping expects {groups.channels}")
    halo = groups.filter_len - 1
    if local.shape[-1] < halo:
        raise ValueError(f"shard length {local.shape[-1]} shorter than halo {halo}")
    for r in range(grp.n_ranks):
        grp.filter_elements[r] = groups.n_groups * groups.filter_len  # full bank everywhere
    return halo


def _exchange_halo(local: torch.Tensor, halo: int, grp: CPGroup, scheme: str):
    """Start the send of the last `halo` steps to rank r+1 and the receive from r-1."""
    n, r = grp.n_ranks, grp.rank
    chans = int(np.prod(local.shape[:-1]))
    for src in range(n - 1):  # every rank tallies the N-1 boundary messages
        grp._send(scheme, src, src + 1, chans * halo)
    left = torch.zeros(local.shape[:-1] + (halo,), dtype=local.dtype, device=local.device)
    ops_ = []
    if r < n - 1:
        ops_.append(("send", local[..., local.shape[-1] - halo:].contiguous(), r + 1))
    if r > 0:
        ops_.append(("recv", left, r - 1))
    return left, _batch_p2p(grp, ops_)


def p2p_conv(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, layout: str = "sequential",
             conv=None) -> torch.Tensor:
    """Halo exchange, then the conv over [halo | local] minus the first halo outputs."""
    halo = _check_p2p(local, groups, grp, layout)
    if halo == 0:
        return (conv or _gpu_conv(_taps_tensor(groups, local), groups.group_size))(local)
    left, reqs = _exchange_halo(local, halo, grp, "p2p_conv")
    for q in reqs:
        q.wait()
    conv = conv or _gpu_conv(_taps_tensor(groups, local), groups.group_size)
    return conv(torch.cat([left, local], dim=-1))[..., halo:].contiguous()


def p2p_conv_overlapped(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, layout: str = "sequential",
                        conv=None, correct=None) -> torch.Tensor:
    """Local conv on zero history first (overlapping the halo transfer), then the correction
    conv([halo | 0])[:, halo:] added to the first halo outputs (cpsim.py:498-510)."""
    halo = _check_p2p(local, groups, grp, layout)
    taps = None
    if conv is None or correct is None:
        taps = _taps_tensor(groups, local)
    conv = conv or _gpu_conv(taps, groups.group_size)
    if halo == 0:
        return conv(local)
    left, reqs = _exchange_halo(local, halo, grp, "p2p_conv_overlapped")
    y = conv(local)  # issued before the halo is consumed
    for q in reqs:
        q.wait()
    if grp.rank > 0:
        y = (correct or _gpu_correct(taps, groups.group_size))(left, y)
    return y


# ---------------------------------------------------------------- all-to-all schemes


def _slab_groups(groups: GroupSpec, start: int, count: int) -> GroupSpec:
    """Sub-bank for a channel slab; slab edges must respect groups (cpsim.py:325-333)."""
    if start % groups.group_size != 0 or count % groups.group_size != 0:
        raise ValueError(f"channel slab [{start}, {start + count}) splits a filter group of size {groups.group_size}")
    first = start // groups.group_size
    return GroupSpec(count, groups.group_size, groups.filters[first:first + count // groups.group_size])


def _a2a(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, n_pipe: int, layout: str, scheme: str,
         conv_slab) -> torch.Tensor:
    n, r = grp.n_ranks, grp.rank
    if local.dim() != 2:
        raise ValueError("all-to-all schemes take the rank's (C, L/N) shard")
    d, m = local.shape
    if d != groups.channels:
        raise ValueError(f"input has {d} channels, grouping expects {groups.channels}")
    if d % n != 0:
        raise ValueError(f"channel count {d} not divisible by {n} ranks")
    if (d // n) % n_pipe != 0:
        raise ValueError(f"per-rank slab {d // n} not divisible by {n_pipe} pipeline segments")
    seg = d // n_pipe
    slab = seg // n
    for s in range(n_pipe):
        for rr in range(n):
            _slab_groups(groups, s * seg + rr * slab, slab)
    for rr in range(n):
        grp.filter_elements[rr] = sum(_slab_groups(groups, s * seg + rr * slab, slab).n_groups
                                      for s in range(n_pipe)) * groups.filter_len
    segmented = getattr(conv_slab, "segmented", False) and layout == "sequential"
    cols = None if segmented else torch.from_numpy(natural_cols(layout, n, m * n)).to(local.device)
    out = torch.empty_like(local)
    for s in range(n_pipe):
        lo = s * seg
        for src in range(n):  # scatter round: every rank sends N-1 slab pieces
            for dst in range(n):
                if dst != src:
                    grp._send(scheme, src, dst, slab * m)
        recv = torch.empty((n, slab, m), dtype=local.dtype, device=local.device)
        _all_to_all(grp, recv, local[lo:lo + seg].contiguous())
        if segmented:
            # recv[src, c] is time segment src of slab row c: the conv reads and writes this
            # rank-major layout directly, and its output is already the return send buffer
            back = conv_slab(recv, _slab_groups(groups, lo + r * slab, slab))
        else:
            assembled = recv.permute(1, 0, 2).reshape(slab, n * m)  # rank-major time order
            natural = torch.empty_like(assembled)
            natural[:, cols] = assembled
            result = conv_slab(natural, _slab_groups(groups, lo + r * slab, slab))
            back = result[:, cols].reshape(slab, n, m).permute(1, 0, 2).contiguous()  # (dst, slab, m)
        for src in range(n):  # return round
            for dst in range(n):
                if dst != src:
                    grp._send(scheme, src, dst, slab * m)
        if n_pipe == 1:
            _all_to_all(grp, out.view(n, slab, m), back)
        else:
            ret = torch.empty((n, slab, m), dtype=local.dtype, device=local.device)
            _all_to_all(grp, ret, back)
            out[lo:lo + seg] = ret.reshape(seg, m)
    grp.count_rounds(scheme, 2 * n_pipe)
    return out


def _gpu_slab_conv(natural: torch.Tensor, bank: GroupSpec) -> torch.Tensor:
    return _gpu_conv(_taps_tensor(bank, natural), bank.group_size)(natural)


def a2a_conv(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, layout: str = "sequential",
             conv_slab=None) -> torch.Tensor:
    """Time shard -> channel slab, conv over the full sequence, back (cpsim.py:428-437)."""
    return _a2a(local, groups, grp, 1, layout, "a2a_conv", conv_slab or _gpu_slab_conv)


@dataclass
class A2ASaved:
    """Forward context of the all-to-all scheme (cpsim.py:421-425)."""

    groups: GroupSpec
    layout: str
    n_ranks: int


def a2a_conv_saved(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, layout: str = "sequential",
                   conv_slab=None):
    """(y shard, A2ASaved) (cpsim.py:433-437)."""
    return a2a_conv(local, groups, grp, layout, conv_slab), A2ASaved(groups, layout, grp.n_ranks)


def _gpu_slab_backward(natural: torch.Tensor, bank: GroupSpec) -> torch.Tensor:
    """Input adjoint of the slab conv (cpsim.py:417-418): dx[t] = sum_j h[j] dy[t+j]."""
    from .ops import causal_conv_bwd
    dx, _ = causal_conv_bwd(natural.contiguous(), None, _taps_tensor(bank, natural), bank.group_size,
                            want_dtaps=False)
    return dx


def a2a_conv_backward(saved: A2ASaved, dy_local: torch.Tensor, grp: CPGroup, layout: str | None = None,
                      conv_slab=None) -> torch.Tensor:
    """Input gradients via two more all-to-all rounds, the correlation on the channel slab
    (cpsim.py:440-446); accounted under the forward's "a2a_conv" scheme like the reference."""
    if not isinstance(saved, A2ASaved):
        raise ValueError("backward needs the A2ASaved context from a2a_conv_saved")
    if grp.n_ranks != saved.n_ranks or (layout is not None and layout != saved.layout):
        raise ValueError("gradient sharding does not match the forward sharding")
    return _a2a(dy_local, saved.groups, grp, 1, saved.layout, "a2a_conv", conv_slab or _gpu_slab_backward)


def a2a_conv_pipelined(local: torch.Tensor, groups: GroupSpec, grp: CPGroup, n_pipe: int,
                       layout: str = "sequential", conv_slab=None) -> torch.Tensor:
    """The a2a scheme in n_pipe channel segments (cpsim.py:449-454)."""
    if n_pipe < 1:
        raise ValueError(f"n_pipe must be >= 1, got {n_pipe}")
    return _a2a(local, groups, grp, n_pipe, layout, "a2a_conv_pipelined", conv_slab or _gpu_slab_conv)


# ---------------------------------------------------------------- context-parallel Hyena operator


# ---------------------------------------------------------------- distributed FFT (cpsim.py:537-659)


def _partner_exchange(x: torch.Tensor, partner: int, grp: CPGroup) -> torch.Tensor:
    """Swap a complex tensor with one partner rank (both send, both receive)."""
    xr = torch.view_as_real(x).contiguous()
    out = torch.empty_like(xr)
    reqs = _batch_p2p(grp, [("send", xr, partner), ("recv", out, partner)])
    for q in reqs:
        q.wait()
    return torch.view_as_complex(out)


def _dfft_check(local: torch.Tensor, grp: CPGroup) -> int:
    from .fft import require_pow2
    require_pow2(local.shape[-1])
    return local.shape[-1]


def _complex(local: torch.Tensor) -> torch.Tensor:
    if local.is_complex():
        return local
    return local.to(torch.complex128 if local.dtype == torch.float64 else torch.complex64)


def _stage_twiddle(g: int, half: int, m: int, length: int, sign: float, like: torch.Tensor) -> torch.Tensor:
    pos = torch.arange(m, dtype=torch.float64) + (g if g < half else g - half) * m
    ang = sign * 2.0 * np.pi * pos / length
    return torch.polar(torch.ones_like(ang), ang).to(like.device, like.dtype)


def _local_fft(x: torch.Tensor, inverse: bool) -> torch.Tensor:
    """The per-rank transform after the cross-rank stages: the hand-written Stockham kernel on
    device tensors (hy_fft_c2c); host tensors (the gloo CPU tests of the scheme's host logic)
    use torch.fft."""
    if x.is_cuda:
        from .ops import fft_c2c
        return fft_c2c(x, inverse=inverse)
    return torch.fft.ifft(x) if inverse else torch.fft.fft(x)


def p2p_fft_forward(local: torch.Tensor, grp: CPGroup, scheme: str = "p2p_fft_conv") -> torch.Tensor:
    """This rank's spectrum slice of the sequentially sharded signal (cpsim.py:547-566, 596-604):
    stage s pairs rank r with r +- half inside groups of N >> (s-1) ranks; the low half keeps
    x + other, the high half (other - x) * W^pos; then a local FFT. Rank r ends up owning the
    bins congruent to bitrev(r) mod N."""
    m = _dfft_check(local, grp)
    n, r = grp.n_ranks, grp.rank
    total = m * n
    x = _complex(local)
    elems = int(x.numel())
    grp.note_resident(r, m)
    stages = int(np.log2(n))
    for stage in range(1, stages + 1):
        group, length = n >> (stage - 1), total >> (stage - 1)
        half = group // 2
        g = r % group
        for src in range(n):  # every rank tallies every message
            gs_ = src % group
            grp._send(scheme, src, src + half if gs_ < half else src - half, elems)
        partner = r + half if g < half else r - half
        other = _partner_exchange(x, partner, grp)
        if g < half:
            x = x + other
        else:
            x = (other - x) * _stage_twiddle(g, half, m, length, -1.0, x)
        grp.note_resident(r, m)
    grp.count_rounds(scheme, stages)
    return _local_fft(x, inverse=False)


def p2p_fft_inverse(spec: torch.Tensor, grp: CPGroup, scheme: str = "p2p_fft_conv") -> torch.Tensor:
    """Inverse of p2p_fft_forward (cpsim.py:569-590, 607-615): local inverse FFT, then the
    stages in reverse with conjugate twiddles and a factor 1/2; restores the sequential shard."""
    n, r = grp.n_ranks, grp.rank
    x = _local_fft(spec, inverse=True)
    m = x.shape[-1]
    total = m * n
    elems = int(x.numel())
    grp.note_resident(r, m)
    stages = int(np.log2(n))
    for stage in range(stages, 0, -1):
        group, length = n >> (stage - 1), total >> (stage - 1)
        half = group // 2
        g = r % group
        for src in range(n):
            gs_ = src % group
            grp._send(scheme, src, src + half if gs_ < half else src - half, elems)
        partner = r + half if g < half else r - half
        other = _partner_exchange(x, partner, grp)
        w_inv = _stage_twiddle(g, half, m, length, 1.0, x)
        x = 0.5 * (x + w_inv * other) if g < half else 0.5 * (other - w_inv * x)
        grp.note_resident(r, m)
    grp.count_rounds(scheme, stages)
    return x


def p2p_fft_conv(local_x: torch.Tensor, local_h: torch.Tensor, grp: CPGroup) -> torch.Tensor:
    """Circular convolution with both operands sharded along time (cpsim.py:618-631)."""
    _dfft_check(local_x, grp)
    _dfft_check(local_h, grp)
    if tuple(local_h.shape) != tuple(local_x.shape):
        raise ValueError("filter must be sharded identically to the input")
    for r in range(grp.n_ranks):
        grp.filter_elements[r] = int(local_h.numel())
    prod = p2p_fft_forward(local_x, grp) * p2p_fft_forward(local_h, grp)
    return p2p_fft_inverse(prod, grp).real.contiguous()


def p2p_fft_causal_wrapper(x: SeqTensor, h_taps, grp: CPGroup | None = None, device=None) -> SeqTensor:
    """Causal linear convolution on the distributed circular core (cpsim.py:634-659): pad to
    2 * next_pow2(L), each rank takes its sequential shard of the padded signal and filter,
    runs p2p_fft_conv, and the shards are gathered and truncated. Every rank returns y."""
    from .fft import next_pow2
    grp = grp or CPGroup()
    taps = np.asarray(h_taps, dtype=np.float64)
    if taps.ndim == 1:
        taps = np.broadcast_to(taps, (x.channels, taps.size))
    if taps.shape[0] != x.channels:
        raise ValueError(f"taps cover {taps.shape[0]} channels, input has {x.channels}")
    taps = taps[:, : x.length]
    size = 2 * next_pow2(x.length)
    n, r = grp.n_ranks, grp.rank
    m = size // n
    dev = device if device is not None else ("cuda" if dist.get_backend(grp.group) == "nccl" else "cpu")
    xp = np.zeros((x.channels, size))
    xp[:, : x.length] = x.data
    hp = np.zeros((x.channels, size))
    hp[:, : taps.shape[1]] = taps
    lx = torch.from_numpy(np.ascontiguousarray(xp[:, r * m:(r + 1) * m])).to(dev)
    lh = torch.from_numpy(np.ascontiguousarray(hp[:, r * m:(r + 1) * m])).to(dev)
    y_local = p2p_fft_conv(lx, lh, grp)
    parts = [torch.empty_like(y_local) for _ in range(n)]
    _all_gather(grp, parts, y_local)
    y = torch.cat(parts, dim=-1)[:, : x.length].cpu().numpy()
    return SeqTensor(y, dtype=x.dtype)


class HyenaCP:
    """Context-parallel Hyena operator: each rank holds the (B, D, L/N) time
    shard of x (sequential layout) and returns its shard of y.

    * projections, gates and the output projection are token-local (no communication);
    * SE / MR (fused tcgen05 mixer): one p2p round ships the last HY_MIXER_HISTORY = 144
      steps of the projections (3D rows) to rank r+1, which the mixer reads as the history
      before its t = 0 (the featurizer halo and the inner-conv halo in one message);
    * LI and the unfused paths: featurizer halo (lhf-1 steps of the projections) by the
      overlapped p2p scheme, then u = k*v either by the overlapped p2p halo (lh-1 steps)
      or, for LI, by the two all-to-all rounds to channel slabs and back.
    """

    def __init__(self, cfg, dtype: torch.dtype = torch.bfloat16, grp: CPGroup | None = None, n_pipe: int | None = None,
                 layout: str = "sequential"):
        from .hyena import HyenaOperator
        if layout not in LAYOUTS:
            raise ValueError(f"layout must be one of {LAYOUTS}, got {layout!r}")
        self.op = HyenaOperator(cfg, dtype)
        self.cfg = cfg
        self.grp = grp or CPGroup()
        self.layout = layout
        # LI: channel segments pipelined through the all-to-all
        self.n_pipe = n_pipe if n_pipe is not None else int(os.environ.get("HY_CP_NPIPE", "4"))

    def _halo_peer(self, tail: torch.Tensor):
        """The group's PeerHalo for this tail shape (CUDA devices only)."""
        return self.grp.peer("halo", tail.shape, tail.dtype) if tail.is_cuda else None

    def _fused(self, m: int) -> bool:
        """The tcgen05 mixer with a projection history (the only mixer that takes one): bf16,
        lh <= 129, rows of m % 8 == 0 (hy_hyena_mixer_fwd's routing rule)."""
        return self.op.dtype == torch.bfloat16 and self.op.lh <= 129 and self.cfg.variant != "LI" and m % 8 == 0

    def _li_pipelined(self, m: int) -> bool:
        op, n = self.op, self.grp.n_ranks
        return (self.cfg.variant == "LI" and op.li_modes is not None and op.lhf <= 8 and m % 4096 == 0
                and self.n_pipe >= 1 and self.cfg.width % (self.n_pipe * n) == 0
                and (self.cfg.width // (self.n_pipe * n)) % self.cfg.inner.group_size == 0)

    def _li_segments(self):
        """Per channel segment: the [q; k; v] rows of W_qkv^T, the featurizer taps and the
        (residues, poles) of every rank's slab, reordered once."""
        if getattr(self, "_segs", None) is not None:
            return self._segs
        op, n = self.op, self.grp.n_ranks
        D = self.cfg.width
        seg = D // self.n_pipe
        segs = []
        for s in range(self.n_pipe):
            rows = torch.cat([torch.arange(i * D + s * seg, i * D + (s + 1) * seg) for i in range(3)]).to(op.dev)
            w = op.w_qkv_t.index_select(0, rows).contiguous()
            wp = None
            if op.split3:
                wp = blas.Split3(tuple(p.index_select(0, rows).contiguous() for p in op.w_qkv_parts))
                wp.cat = op.w_qkv_parts.cat.index_select(0, rows).contiguous()
            ft = op.feat_taps[:, s * seg:(s + 1) * seg].contiguous()
            g0 = (s * seg + self.grp.rank * (seg // n)) // op.gs
            ng = (seg // n) // op.gs
            res, poles = (t[g0:g0 + ng].contiguous() for t in op.li_modes)
            segs.append((rows, w, wp, ft, res, poles))
        self._segs = segs
        return segs

    def _li_pipeline(self, x3: torch.Tensor, events=None) -> torch.Tensor:
        """LI layer in n_pipe channel segments (the reference's a2a_conv_pipelined, cpsim.py:449-454,
        taken up to the projections): segment s's projection GEMM and featurizer stream run on the
        compute stream while segment s-1's all-to-all rounds and slab conv run on a side stream, so
        the NVLink traffic hides behind the GEMMs. The all-to-all rounds are copy-engine copies into
        the peers' symmetric buffers over NVLink (p2p.PeerAllToAll; HY_CP_P2P=0 selects NCCL's
        all_to_all_single). The featurizer halo (the predecessor's last 8
        raw projected steps of every row) comes first from a small GEMM on the last 8 input steps
        and one p2p round."""
        from . import ops
        op, grp = self.op, self.grp
        n, r = grp.n_ranks, grp.rank
        B, D, m = x3.shape
        seg = D // self.n_pipe
        slab = seg // n
        segs = self._li_segments()
        comp = torch.cuda.current_stream()
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream(device=x3.device)
        comm = self._comm
        peer = None
        if os.environ.get("HY_CP_P2P", "1") != "0":
            # two segments in flight (scatter of s while s-1 is convolved): 2 B slots, so no
            # slot is rewritten while a use of it is still being read
            peer = grp.peer("a2a", (slab, m), x3.dtype, 2 * B)
        tail = op.project(x3[..., m - 8:].contiguous())  # (B, 3D, 8)
        hpeer = self._halo_peer(tail) if peer is not None else None
        if hpeer is not None:
            hk = hpeer.next_slot()
            for src in range(n - 1):
                grp._send("cp_feat_hist", src, src + 1, tail.numel())
            hist = hpeer.send(tail, hk)
            hpeer.wait(hk)
        else:
            hist, reqs = _exchange_halo(tail, 8, grp, "cp_feat_hist")
            for q in reqs:
                q.wait()
        mixed = torch.empty((B, D, m), dtype=x3.dtype, device=x3.device)
        for r_ in range(n):
            grp.filter_elements[r_] = self.cfg.inner.n_groups // n * self.cfg.inner.filter_len
        if peer is not None and os.environ.get("HY_CP_LI_SCHED", "serial") == "serial":
            self._li_serial(x3, segs, hist, peer, mixed, events)
            grp.count_rounds("a2a_conv_pipelined", 2 * self.n_pipe * B)
            hpeer.release(hk)
            return mixed
        pending = []
        for s, (rows, w, wp, ft, res, poles) in enumerate(segs):
            proj_s = blas.matmul_split3(wp, blas.split3_act(x3)) if op.split3 else torch.matmul(w, x3)
            rh = hist.index_select(1, rows).contiguous() if r > 0 else None
            u_s, fq_s = ops.featurize(proj_s, ft, rhist=rh)
            ev = torch.cuda.Event()
            ev.record(comp)
            with torch.cuda.stream(comm):
                comm.wait_event(ev)
                for b in range(B):
                    for src in range(n):  # the reference's accounting: scatter + return rounds
                        for dst in range(n):
                            if dst != src:
                                grp._send("a2a_conv_pipelined", src, dst, 2 * slab * m)
                    if peer is not None:  # copy engines over NVLink peer memory
                        k = peer[0].next_slot()
                        recv = peer[0].exchange(u_s[b].view(n, slab, m), k)
                    else:
                        recv = torch.empty((n, slab, m), dtype=x3.dtype, device=x3.device)
                        _all_to_all(grp, recv, u_s[b])
                    if events is not None and s == 0 and b == 0:
                        events[0].record(comm)
                    y_slab = ops.li_conv_segmented(recv, res, poles, op.gs)
                    if events is not None and s == 0 and b == 0:
                        events[1].record(comm)
                    if peer is not None:
                        peer[0].release(k)
                        back = peer[1].exchange(y_slab, k)
                    else:
                        back = torch.empty((n, slab, m), dtype=x3.dtype, device=x3.device)
                        _all_to_all(grp, back, y_slab)
                    ops.gate_mul(fq_s[b], back.view(seg, m), out=mixed[b, s * seg:(s + 1) * seg])
                    if peer is not None:
                        peer[1].release(k)
                u_s.record_stream(comm)
                fq_s.record_stream(comm)
            pending.append(u_s)
        grp.count_rounds("a2a_conv_pipelined", 2 * self.n_pipe * B)
        if hpeer is not None:  # every segment's featurizer stream has read the history
            hpeer.release(hk)
        comp.wait_stream(comm)
        return mixed

    def _li_serial(self, x3, segs, hist, peer, mixed, events=None):
        """The LI layer as a software pipeline on ONE compute stream, the all-to-all rounds on
        the copy engines: iteration s runs segment s's projection GEMM and featurizer stream and
        starts its scatter copies, then segment s-1's slab conv (its scatter landed during
        GEMM s) and the start of its return copies, then segment s-2's gating (its return
        landed during GEMM s). No kernel shares the SMs with the GEMMs, and no stream waits on
        copies issued after it."""
        from . import ops
        op, grp = self.op, self.grp
        n, r = grp.n_ranks, grp.rank
        B, D, m = x3.shape
        seg = D // self.n_pipe
        slab = seg // n
        live = {}  # s -> (fq_s, scatter slots, return slots)

        def start(s):
            rows, w, wp, ft, _, _ = segs[s]
            proj_s = blas.matmul_split3(wp, blas.split3_act(x3)) if op.split3 else torch.matmul(w, x3)
            rh = hist.index_select(1, rows).contiguous() if r > 0 else None
            u_s, fq_s = ops.featurize(proj_s, ft, rhist=rh)
            ks = []
            for b in range(B):
                for src in range(n):  # the reference's accounting: scatter + return rounds
                    for dst in range(n):
                        if dst != src:
                            grp._send("a2a_conv_pipelined", src, dst, 2 * slab * m)
                k = peer[0].next_slot()
                ks.append((k, peer[0].send(u_s[b].view(n, slab, m), k)))
            live[s] = (fq_s, ks, [])

        def conv(s):
            _, _, _, _, res, poles = segs[s]
            fq_s, ks, kb = live[s]
            for b in range(B):
                recv = peer[0].wait(*ks[b])  # this use of the slot (later sends may share it)
                if events is not None and s == 0 and b == 0:
                    events[0].record()
                y_slab = ops.li_conv_segmented(recv, res, poles, op.gs)
                if events is not None and s == 0 and b == 0:
                    events[1].record()
                peer[0].release(*ks[b])
                k = peer[1].next_slot()
                kb.append((k, peer[1].send(y_slab, k)))

        def gate(s):
            fq_s, _, kb = live.pop(s)
            for b in range(B):
                back = peer[1].wait(*kb[b])
                ops.gate_mul(fq_s[b], back.view(seg, m), out=mixed[b, s * seg:(s + 1) * seg])
                peer[1].release(*kb[b])

        for it in range(self.n_pipe + 2):
            if it < self.n_pipe:
                start(it)
            if 1 <= it <= self.n_pipe:
                conv(it - 1)
            if it >= 2:
                gate(it - 2)

    def forward(self, x_local: torch.Tensor, events=None, accumulate_into: torch.Tensor | None = None) -> torch.Tensor:
        """events: optional (start, end) CUDA events recorded around the mixer / local conv.
        accumulate_into: caller-owned tensor the output is added into in the out-projection
        GEMM epilogue (residual stacks; see HyenaOperator.forward)."""
        from . import _lib, ops
        op, grp = self.op, self.grp
        if grp.n_ranks == 1:  # one rank: the whole sequence is local, the fused operator applies
            return op.forward(x_local, events=events, accumulate_into=accumulate_into)
        if self.layout == "zigzag":
            return self._forward_zigzag(x_local, events, accumulate_into)
        x3 = x_local.unsqueeze(0) if x_local.dim() == 2 else x_local
        B, D, m = x3.shape
        if self._fused(m) and m >= _lib.MIXER_HISTORY:
            # the successor needs only the projections of the last 144 steps: compute those
            # first and start the send, so the transfer overlaps the full projection GEMM
            tail = op.project(x3[..., m - _lib.MIXER_HISTORY:].contiguous())
            peer = self._halo_peer(tail) if os.environ.get("HY_CP_P2P", "1") != "0" else None
            if peer is not None:  # copy engine into rank r+1's symmetric slot (no SMs, no NCCL)
                k = peer.next_slot()
                for src in range(grp.n_ranks - 1):
                    grp._send("cp_hist", src, src + 1, tail.numel() // tail.shape[-1] * _lib.MIXER_HISTORY)
                hist = peer.send(tail, k)
                proj = op.project(x3)  # (B, 3D, m): token-local
                peer.wait(k)
            else:
                hist, reqs = _exchange_halo(tail, _lib.MIXER_HISTORY, grp, "cp_hist")
                proj = op.project(x3)  # (B, 3D, m): token-local
                for q in reqs:
                    q.wait()
            if events is not None:
                events[0].record()
            mixed = ops.hyena_mixer(proj, op.feat_taps, op.inner_taps, op.gs, decay=op.decay,
                                    packed=op.feat_packed, hist=hist if grp.rank > 0 else None)
            if peer is not None:
                peer.release(k)
            if events is not None:
                events[1].record()
        elif self._li_pipelined(m):
            mixed = self._li_pipeline(x3, events)
        else:
            proj = op.project(x3)  # (B, 3D, m): token-local
            # featurizers over the 3D projected rows with their (lhf-1)-step halo
            ft = op.feat_taps.reshape(3 * D, op.lhf)
            if getattr(self, "_feat_groups", None) is None:
                self._feat_groups = _per_channel_groups(ft)
            feat_groups = self._feat_groups
            feats = p2p_conv_overlapped(proj, feat_groups, grp,
                                        conv=lambda z: ops.causal_conv(z.contiguous(), ft, 1),
                                        correct=lambda h, y: _correct(h, y, ft, 1))
            q, k, v = (feats[:, i * D:(i + 1) * D].contiguous() for i in range(3))
            u = k * v
            taps = op.materialized_inner
            if self.cfg.variant == "LI":
                m = u.shape[-1]
                if op.li_modes is not None and m % 4096 == 0:
                    slab_conv = _li_slab_conv(op, events)
                elif op.li_scan_modes is not None:
                    slab_conv = _li_scan_slab_conv(op)
                else:
                    slab_conv = None  # materialised taps, direct conv on the natural-order slab
                conv = torch.stack([a2a_conv(u[b].contiguous(), self.cfg.inner, grp, conv_slab=slab_conv)
                                    for b in range(B)])
            else:
                conv = p2p_conv_overlapped(u, self.cfg.inner, grp,
                                           conv=lambda z: ops.gated_conv(z.contiguous(), taps, op.gs),
                                           correct=lambda h, y: _correct(h, y, taps, op.gs))
            mixed = ops.gate_mul(q, conv.contiguous())
        acc = None
        if accumulate_into is not None:
            acc = accumulate_into.unsqueeze(0) if x_local.dim() == 2 else accumulate_into
        y = op.out_project(mixed, acc)
        return y[0] if x_local.dim() == 2 else y

    __call__ = forward


    # ------------------------------------------------------------ zigzag layout (cpsim.py:282-319)
    def _forward_zigzag(self, x_local: torch.Tensor, events=None, accumulate_into=None) -> torch.Tensor:
        """Rank r holds chunks r and 2N-1-r of the sequence ([half A | half B] in local time).
        Both halves run as one batch of 2B through the token-local projections and the mixers;
        each half's causal history comes from the rank holding its predecessor chunk
        (_zigzag_history): half A from rank r-1's half A, half B from rank r+1's half B (rank
        N-1's half B continues its own half A). The LI long conv uses the zigzag all-to-all."""
        from . import _lib, ops
        op, grp = self.op, self.grp
        x3 = x_local.unsqueeze(0) if x_local.dim() == 2 else x_local
        B, D, m = x3.shape
        if m % 2:
            raise ValueError(f"zigzag shard length {m} is not two equal chunks")
        h = m // 2
        halves = (x3[..., :h], x3[..., h:])
        ft = op.feat_taps
        if self._fused(h) and h >= _lib.MIXER_HISTORY:
            H = _lib.MIXER_HISTORY
            tails = op.project(torch.cat([halves[0][..., h - H:], halves[1][..., h - H:]], dim=0).contiguous())
            hist = _zigzag_history(tails[:B], tails[B:], grp, "cp_zigzag_hist")
            proj = torch.cat([op.project(halves[0].contiguous()), op.project(halves[1].contiguous())], dim=0)
            if events is not None:
                events[0].record()
            mixed = ops.hyena_mixer(proj, ft, op.inner_taps, op.gs, decay=op.decay, packed=op.feat_packed, hist=hist)
            if events is not None:
                events[1].record()
        else:
            if op.lhf > 8:
                raise NotImplementedError("zigzag context parallel needs featurizers of <= 8 taps")
            proj = torch.cat([op.project(halves[0].contiguous()), op.project(halves[1].contiguous())], dim=0)
            rh = _zigzag_history(proj[:B, :, h - 8:].contiguous(), proj[B:, :, h - 8:].contiguous(), grp,
                                 "cp_zigzag_feat")
            u, fq = ops.featurize(proj, ft, rhist=rh)  # (2B, D, h) each
            if self.cfg.variant == "LI":
                slab = self._zigzag_slab_conv()
                u_local = torch.cat([u[:B], u[B:]], dim=-1)  # (B, D, m): the rank's zigzag shard
                conv = torch.stack([a2a_conv(u_local[b].contiguous(), self.cfg.inner, grp, "zigzag", conv_slab=slab)
                                    for b in range(B)])
                conv = torch.cat([conv[..., :h], conv[..., h:]], dim=0)
            else:
                lh = op.lh
                taps = op.materialized_inner
                uh = _zigzag_history(u[:B, :, h - (lh - 1):].contiguous(), u[B:, :, h - (lh - 1):].contiguous(), grp,
                                     "cp_zigzag_inner") if lh > 1 else None
                ext = torch.cat([uh, u], dim=-1) if uh is not None else u
                conv = (ops.long_conv(ext.contiguous(), taps, op.gs) if lh > 129
                        else ops.gated_conv(ext.contiguous(), taps, op.gs))[..., lh - 1:]
            mixed = ops.gate_mul(fq, conv.contiguous())
        if accumulate_into is not None and not op.split3:
            # residual stacks: each half's out projection accumulates into its strided view of the
            # caller's buffer inside the GEMM (cuBLAS beta = 1, ldc = m), as the sequential layout
            acc = accumulate_into.unsqueeze(0) if x_local.dim() == 2 else accumulate_into
            for i in range(2):
                for b in range(B):
                    acc[b, :, i * h:(i + 1) * h].addmm_(op.w_out_t, mixed[i * B + b])
            return acc[0] if x_local.dim() == 2 else acc
        y2 = op.out_project(mixed)  # (2B, D, h)
        y = torch.cat([y2[:B], y2[B:]], dim=-1)
        if accumulate_into is not None:
            acc = accumulate_into.unsqueeze(0) if x_local.dim() == 2 else accumulate_into
            acc.add_(y)
            y = acc
        return y[0] if x_local.dim() == 2 else y

    def _zigzag_slab_conv(self):
        """Natural-order slab conv for the zigzag all-to-all: the implicit filter's tcgen05
        kernel (bf16, <= 8 poles, L % 8 == 0) or the modal scan, else the materialised taps."""
        from . import ops
        op = self.op
        if op.li_modes is not None:
            res, poles = op.li_modes

            def conv(natural, slab_groups):
                g0 = _group_index(op.cfg.inner, slab_groups)
                ng = slab_groups.n_groups
                if natural.shape[-1] % 8 == 0:
                    return ops.li_conv(natural.contiguous(), res[g0:g0 + ng], poles[g0:g0 + ng], slab_groups.group_size)
                return ops.li_scan(natural.contiguous(), op.li_scan_modes[0][g0:g0 + ng],
                                   op.li_scan_modes[1][g0:g0 + ng], slab_groups.group_size)
            return conv
        if op.li_scan_modes is not None:
            return _li_scan_slab_conv(op)
        return None


def _zigzag_history(tail_a: torch.Tensor, tail_b: torch.Tensor, grp: CPGroup, scheme: str) -> torch.Tensor:
    """Causal histories of a zigzag shard's two halves (cpsim.py:282-319 layout; rank r holds
    chunks r and 2N-1-r): half A's predecessor chunk r-1 is rank r-1's half A (rank 0: none,
    zeros); half B's predecessor chunk 2N-2-r is rank r+1's half B, except on rank N-1, whose
    half B (chunk N) continues its own half A (chunk N-1). tail_a / tail_b: this rank's last
    steps of each half, (B, C, H). Returns (2B, C, H) = [history of A; history of B]."""
    n, r = grp.n_ranks, grp.rank
    chans = int(np.prod(tail_a.shape[:-1]))
    for src in range(n - 1):  # every rank tallies every message: A tails go up, B tails go down
        grp._send(scheme, src, src + 1, chans * tail_a.shape[-1])
        grp._send(scheme, src + 1, src, chans * tail_b.shape[-1])
    hist_a = torch.zeros_like(tail_a)
    hist_b = tail_a.clone() if r == n - 1 else torch.empty_like(tail_b)
    ops_ = []
    if r < n - 1:
        ops_.append(("send", tail_a.contiguous(), r + 1))
        ops_.append(("recv", hist_b, r + 1))
    if r > 0:
        ops_.append(("send", tail_b.contiguous(), r - 1))
        ops_.append(("recv", hist_a, r - 1))
    for q in _batch_p2p(grp, ops_):
        q.wait()
    grp.count_rounds(scheme, 1)
    return torch.cat([hist_a, hist_b], dim=0).contiguous()


def _li_slab_conv(op, events=None):
    """Implicit long conv of a channel slab over the full sequence, read and written in the
    rank-major all-to-all layout (tcgen05 li_conv_segmented); events: optional (start, end)
    CUDA events around the kernel."""
    from . import ops
    res, poles = op.li_modes

    def conv(recv, slab_groups):
        g0 = _group_index(op.cfg.inner, slab_groups)
        ng = slab_groups.n_groups
        if events is not None:
            events[0].record()
        y = ops.li_conv_segmented(recv, res[g0:g0 + ng], poles[g0:g0 + ng], slab_groups.group_size)
        if events is not None:
            events[1].record()
        return y
    conv.segmented = True
    return conv


def _li_scan_slab_conv(op):
    """Implicit long conv of a natural-order channel slab by the modal scan (hy_li_scan_fwd:
    fp32 / fp64 slabs, > 8 poles, shards that are not multiples of the tcgen05 tile)."""
    from . import ops
    res, poles = op.li_scan_modes

    def conv(natural, slab_groups):
        g0 = _group_index(op.cfg.inner, slab_groups)
        ng = slab_groups.n_groups
        return ops.li_scan(natural.contiguous(), res[g0:g0 + ng], poles[g0:g0 + ng], slab_groups.group_size)
    return conv


def _group_index(bank: GroupSpec, sub: GroupSpec) -> int:
    first = sub.filters[0]
    for i, f in enumerate(bank.filters):
        if f is first:
            return i
    raise ValueError("slab filters not found in the operator's bank")


def _correct(halo, y, taps, gs):
    from . import ops
    y = y.contiguous()
    ops.halo_correction(halo.contiguous(), y, taps, gs)
    return y


def _per_channel_groups(taps: torch.Tensor) -> GroupSpec:
    from .core import ExplicitFilter
    t = taps.detach().double().cpu().numpy()
    return GroupSpec(t.shape[0], 1, tuple(ExplicitFilter(r) for r in t))


class LayoutCP:
    """Multi-layer context-parallel stack (hyena.py:377-392 over cpsim's
    sequential sharding): the sequence is sharded once, every layer runs as HyenaCP on the
    rank's (B, D, L/N) shard and the residual add is token-local, so activations stay sharded
    from the first layer to the last. Layers share the group's peer buffers (CPGroup.peer)."""

    def __init__(self, stack, dtype: torch.dtype = torch.bfloat16, grp: CPGroup | None = None,
                 n_pipe: int | None = None, layout: str = "sequential"):
        self.grp = grp or CPGroup()
        self.layout = layout
        self.layers = [HyenaCP(cfg, dtype, self.grp, n_pipe, layout) for cfg in stack.layers]
        self.residual = stack.residual

    def forward(self, x_local: torch.Tensor) -> torch.Tensor:
        cur = x_local
        for i, layer in enumerate(self.layers):
            if self.residual:  # residual add fused into the out-projection GEMM epilogue
                cur = layer.forward(cur, accumulate_into=cur.clone() if i == 0 else cur)
            else:
                cur = layer.forward(cur)
        return cur

    __call__ = forward


def layout_forward_cp(x_local: torch.Tensor, stack, grp: CPGroup | None = None,
                      layout: str = "sequential") -> torch.Tensor:
    """layout_forward (hyena.py:386) on this rank's shard of x (sequential or zigzag layout)."""
    return LayoutCP(stack, x_local.dtype, grp, layout=layout).forward(x_local)
