"""Context-parallel conv schemes restated as plain per-rank loops (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/convhybrid/cpsim.py without its generator
fabric: each scheme computes every rank's result directly and tallies the
messages / elements / rounds the reference's SimGroup would log for it
(cpsim.py:97-131). Used to check the torch.distributed CP layer.
"""

from __future__ import annotations

import numpy as np

from .ref import F64, bank_filter_len, direct_causal_conv

LAYOUTS = ("sequential", "zigzag")


class Tally:
    """Counters mirroring SimGroup accounting (cpsim.py:69-131)."""

    def __init__(self, n_ranks: int):
        if n_ranks < 1 or (n_ranks & (n_ranks - 1)) != 0:
            raise ValueError(f"rank count must be a power of two >= 1, got {n_ranks}")
        self.n_ranks = n_ranks
        self.elements: dict = {}
        self.messages: dict = {}
        self.rounds: dict = {}
        self.filter_elements: dict = {}

    def send(self, scheme: str, elements: int) -> None:
        self.elements[scheme] = self.elements.get(scheme, 0) + int(elements)
        self.messages[scheme] = self.messages.get(scheme, 0) + 1


def layout_chunks(layout: str, n_ranks: int):
    """(cpsim.py:282-286)."""
    if layout == "sequential":
        return [[r] for r in range(n_ranks)]
    return [[r, 2 * n_ranks - 1 - r] for r in range(n_ranks)]


def shard(x: np.ndarray, n_ranks: int, layout: str = "sequential"):
    """(cpsim.py:289-301)."""
    if layout not in LAYOUTS:
        raise ValueError(f"layout must be one of {LAYOUTS}, got {layout!r}")
    divisor = n_ranks * (1 if layout == "sequential" else 2)
    if x.shape[1] % divisor != 0:
        raise ValueError(f"length {x.shape[1]} not divisible by {divisor}")
    clen = x.shape[1] // divisor
    return [np.concatenate([x[:, c * clen:(c + 1) * clen] for c in ids], axis=1)
            for ids in layout_chunks(layout, n_ranks)]


def gather(shards, layout: str = "sequential") -> np.ndarray:
    """(cpsim.py:304-312)."""
    n = len(shards)
    ids = layout_chunks(layout, n)
    clen = shards[0].shape[1] // len(ids[0])
    out = np.empty((shards[0].shape[0], shards[0].shape[1] * n), dtype=F64)
    for r, cs in enumerate(ids):
        for i, c in enumerate(cs):
            out[:, c * clen:(c + 1) * clen] = shards[r][:, i * clen:(i + 1) * clen]
    return out


def _slab_bank(bank, start, count):
    """(cpsim.py:325-333)."""
    gs = bank["group_size"]
    if start % gs != 0 or count % gs != 0:
        raise ValueError(f"channel slab [{start}, {start + count}) splits a filter group of size {gs}")
    first = start // gs
    return {"channels": count, "group_size": gs, "filters": bank["filters"][first:first + count // gs]}


def p2p_conv(shards, bank, tally: Tally, overlapped: bool = False):
    """Halo of lh-1 steps from rank r to r+1, then a local conv (cpsim.py:460-534).

    The overlapped form runs the local conv on zero history and adds the
    correction conv([halo || 0])[:, halo:] to the first halo outputs
    (cpsim.py:498-510); both give the same numbers.
    """
    scheme = "p2p_conv_overlapped" if overlapped else "p2p_conv"
    n = len(shards)
    halo = bank_filter_len(bank) - 1
    if shards[0].shape[1] < halo:
        raise ValueError(f"shard length {shards[0].shape[1]} shorter than halo {halo}")
    for r in range(n):
        tally.filter_elements[r] = len(bank["filters"]) * bank_filter_len(bank)
    outs = []
    for r in range(n):
        local = np.asarray(shards[r], dtype=F64)
        d = local.shape[0]
        if halo > 0 and r < n - 1:
            tally.send(scheme, d * halo)
        left = (np.asarray(shards[r - 1], dtype=F64)[:, -halo:] if (halo > 0 and r > 0)
                else np.zeros((d, halo)))
        if not overlapped:
            ext = np.concatenate([left, local], axis=1)
            outs.append(np.asarray(direct_causal_conv(ext, bank), dtype=F64)[:, halo:])
        else:
            y = np.array(direct_causal_conv(local, bank), dtype=F64)
            if halo > 0 and r > 0:
                ov = np.concatenate([left, np.zeros((d, halo))], axis=1)
                y[:, :halo] += np.asarray(direct_causal_conv(ov, bank), dtype=F64)[:, halo:]
            outs.append(y)
    return outs


def a2a_conv(shards, bank, tally: Tally, n_pipe: int = 1, layout: str = "sequential",
             local_conv=None):
    """Time-shard <-> channel-slab swap, conv on the slab, swap back (cpsim.py:336-454).

    ``local_conv(natural_slab, slab_bank)`` defaults to the direct conv the
    reference simulator uses (cpsim.py:413-414).
    """
    scheme = "a2a_conv" if n_pipe == 1 else "a2a_conv_pipelined"
    n = len(shards)
    d, m = shards[0].shape
    if d % n != 0:
        raise ValueError(f"channel count {d} not divisible by {n} ranks")
    if (d // n) % n_pipe != 0:
        raise ValueError(f"per-rank slab {d // n} not divisible by {n_pipe} pipeline segments")
    conv = local_conv or (lambda a, b: np.asarray(direct_causal_conv(a, b), dtype=F64))
    seg = d // n_pipe
    total = m * n
    ids = [c for cs in layout_chunks(layout, n) for c in cs]
    clen = total // len(ids)
    cols = np.concatenate([np.arange(c * clen, (c + 1) * clen) for c in ids])
    outs = [np.empty((d, m)) for _ in range(n)]
    for s in range(n_pipe):
        lo = s * seg
        slab = seg // n
        for r in range(n):
            _slab_bank(bank, lo + r * slab, slab)
        # scatter: every rank sends its time shard of slab dst to dst
        for r in range(n):
            for dst in range(n):
                if dst != r:
                    tally.send(scheme, slab * m)
        for r in range(n):
            assembled = np.concatenate(
                [np.asarray(shards[src], dtype=F64)[lo + r * slab: lo + (r + 1) * slab] for src in range(n)],
                axis=1)
            natural = np.empty_like(assembled)
            natural[:, cols] = assembled
            result = conv(natural, _slab_bank(bank, lo + r * slab, slab))
            back = result[:, cols]
            for dst in range(n):
                if dst != r:
                    tally.send(scheme, slab * m)
                outs[dst][lo + r * slab: lo + (r + 1) * slab] = back[:, dst * m:(dst + 1) * m]
    tally.rounds[scheme] = tally.rounds.get(scheme, 0) + 2 * n_pipe
    for r in range(n):
        tally.filter_elements[r] = sum(
            len(_slab_bank(bank, s * seg + r * (seg // n), seg // n)["filters"]) for s in range(n_pipe)
        ) * bank_filter_len(bank)
    return outs
