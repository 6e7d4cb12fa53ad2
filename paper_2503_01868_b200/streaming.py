"""Host-resident batches through a device forward with copy/compute overlap.

The reference API takes host arrays (`SeqTensor`, core.py:25-60) and returns host arrays;
staged naively, every call serialises H2D copy -> forward -> D2H copy. `HostPipeline`
keeps each step's own copies (step i's inputs go up, step i's result comes back) but runs
them on two copy streams, so the H2D copy of step i+1 and the D2H copy of step i-1 overlap
the forward of step i on the compute stream (the two directions use separate copy engines).
With `chunks > 1` a step's batch is split along its first axis into chunks that go through the
same pipeline (the forward is independent per sequence), so the copies also overlap within a
step and the pipeline's fill and drain shrink to one chunk. At config C2 the host link (PCIe
Gen5 x16, ~50 GB/s per direction with both directions busy, `scripts/pcie_probe.py`) takes
5.4 ms per 268 MB step each way against a 3.0 ms forward, so the e2e rate is the link's; four
chunks per step measured no better on average and much noisier, so the bench streams whole steps.
"""

from __future__ import annotations

import torch


class HostPipeline:
    """fwd(x_device) -> y_device, for pinned host inputs of a fixed shape / dtype."""

    def __init__(self, fwd, shape, dtype: torch.dtype, depth: int = 2, device=None, chunks: int = 1):
        if depth < 2:
            raise ValueError("depth must be >= 2 (double-buffered inputs)")
        if chunks < 1 or shape[0] % chunks:
            raise ValueError(f"chunks ({chunks}) must divide the batch axis ({shape[0]})")
        self.fwd = fwd
        self.depth = depth
        self.chunks = chunks
        dev = device or torch.device("cuda", torch.cuda.current_device())
        cshape = (shape[0] // chunks,) + tuple(shape[1:])
        self.xbuf = [torch.empty(cshape, dtype=dtype, device=dev) for _ in range(depth)]
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.used = [False] * depth

    def run(self, xh, yh, steps: int) -> None:
        """`steps` forwards: each copies its input from host `xh` (a pinned tensor, or a list
        indexed by step) and its result into host `yh` (same convention). Stream-ordered on
        the current stream; synchronise (or record an event after `d2h`) to consume yh."""
        cur = torch.cuda.current_stream()
        nc = self.chunks
        for i in range(steps * nc):
            s = i % self.depth
            step, c = divmod(i, nc)
            src = xh[step % len(xh)] if isinstance(xh, (list, tuple)) else xh
            dst = yh[step % len(yh)] if isinstance(yh, (list, tuple)) else yh
            if nc > 1:
                w = src.shape[0] // nc
                src, dst = src[c * w:(c + 1) * w], dst[c * w:(c + 1) * w]
            buf = self.xbuf[s]
            if self.used[s]:
                self.h2d.wait_event(self.ev_out[s])  # the forward that last read buf is done
            with torch.cuda.stream(self.h2d):
                buf.copy_(src, non_blocking=True)
                self.ev_in[s].record(self.h2d)
            cur.wait_event(self.ev_in[s])
            y = self.fwd(buf)
            self.ev_out[s].record(cur)
            self.used[s] = True
            self.d2h.wait_event(self.ev_out[s])
            with torch.cuda.stream(self.d2h):
                dst.copy_(y, non_blocking=True)
            y.record_stream(self.d2h)
        cur.wait_stream(self.d2h)
        cur.wait_stream(self.h2d)
