"""All-to-all and causal halo over NVLink peer memory for the context-parallel layer (no
NCCL kernels): PeerAllToAll for the LI sequence <-> channel swaps, PeerHalo for the SE/MR
point-to-point history.

Every rank owns a symmetric receive buffer of `nslots` slots, each (n_ranks, chunk) bytes,
allocated with cudaMalloc and mapped into every peer by CUDA IPC (cudaIpcOpenMemHandle with
lazy peer access: the peer's pages are addressed directly over NVLink / NVSwitch). A
transfer is a set of stream-ordered copy-engine copies (cudaMemcpyAsync on peer pointers, one
side stream per destination so the copies run on separate engines and links) followed by a
32-bit flag write into the receiver (cuStreamWriteValue32, with its default memory barrier);
the receiver's stream waits on the flags (cuStreamWaitValue32). The copies take no SMs, so
they overlap the projection GEMMs fully — NCCL's all-to-all kernels would share the SMs.

Flow control per slot: a use counter u. The sender, before writing slot k of rank d for use
u, waits until d has released use u-1 of that slot (d writes u-1 into the sender's `free`
flag after its consumer is enqueued); the receiver waits until every sender's `arrive` flag
reaches u. Nothing is ever host-synchronised.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

try:
    from cuda.bindings import driver as _cu
    from cuda.bindings import runtime as _rt
except ImportError:  # pragma: no cover - cuda-python is part of the image
    _cu = _rt = None

_GEQ = 0  # CU_STREAM_WAIT_VALUE_GEQ
_WDEF = 0  # CU_STREAM_WRITE_VALUE_DEFAULT (fenced)
_D2D = 3  # cudaMemcpyDeviceToDevice


def _ck(res):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"CUDA call failed: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class _RawArray:
    """A cudaMalloc'd region viewed as a torch tensor through __cuda_array_interface__."""

    def __init__(self, ptr: int, shape, dtype: torch.dtype):
        typestr = {torch.bfloat16: "<V2", torch.float32: "<f4", torch.int32: "<i4"}[dtype]
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}
        self.dtype = dtype

    def tensor(self) -> torch.Tensor:
        if self.dtype == torch.bfloat16:  # no bf16 typestr: view 2-byte words as int16 then reinterpret
            iface = dict(self.__cuda_array_interface__, typestr="<i2")
            holder = type("H", (), {"__cuda_array_interface__": iface})()
            return torch.as_tensor(holder, device="cuda").view(torch.bfloat16)
        return torch.as_tensor(self, device="cuda")


class PeerUnavailable(RuntimeError):
    """Raised on every rank when some rank cannot map its peers' buffers."""


class _Symmetric:
    """`nslots` data slots of `slot` bytes plus `nflags` 32-bit flags per rank, cudaMalloc'd
    and mapped into every peer of `group` by CUDA IPC (lazy peer access over NVLink)."""

    def __init__(self, group, slot: int, nslots: int, nflags: int):
        if _rt is None:
            raise RuntimeError("cuda-python is required for the peer-memory transfers")
        self.group = group
        self.n = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.nslots = nslots
        self.slot = slot
        dev = torch.cuda.current_device()
        self.data = int(_ck(_rt.cudaMalloc(nslots * slot)))
        self.flags = int(_ck(_rt.cudaMalloc(nflags * 4)))
        _ck(_rt.cudaMemset(self.flags, 0, nflags * 4))
        _ck(_rt.cudaDeviceSynchronize())
        mine = (bytes(_ck(_rt.cudaIpcGetMemHandle(self.data)).reserved),
                bytes(_ck(_rt.cudaIpcGetMemHandle(self.flags)).reserved), dev)
        allh = [None] * self.n
        dist.all_gather_object(allh, mine, group=group)
        self.peer_data, self.peer_flags = [0] * self.n, [0] * self.n
        self.closed = False
        err = None
        try:
            for p in range(self.n):
                if p == self.r:
                    self.peer_data[p], self.peer_flags[p] = self.data, self.flags
                    continue
                hd, hf = _rt.cudaIpcMemHandle_t(), _rt.cudaIpcMemHandle_t()
                hd.reserved, hf.reserved = allh[p][0], allh[p][1]
                self.peer_data[p] = int(_ck(_rt.cudaIpcOpenMemHandle(hd, _rt.cudaIpcMemLazyEnablePeerAccess)))
                self.peer_flags[p] = int(_ck(_rt.cudaIpcOpenMemHandle(hf, _rt.cudaIpcMemLazyEnablePeerAccess)))
        except RuntimeError as e:  # e.g. no IPC between these processes
            err = e
        # every rank learns whether every rank mapped its peers (no rank may wait alone); the
        # flag travels on the device for NCCL groups, on the host for gloo groups
        on = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=on)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            self._unmap()  # handles opened before the failure, then the local buffers
            self._free_local()
            self.closed = True
            raise PeerUnavailable(f"peer mapping failed on some rank ({err or 'another rank'})")
        self.use = [0] * nslots
        self.step = 0

    def _unmap(self):
        for p in range(self.n):
            for lst in (self.peer_data, self.peer_flags):
                if p != self.r and lst[p]:
                    _rt.cudaIpcCloseMemHandle(lst[p])
                    lst[p] = 0

    def _free_local(self):
        for name in ("data", "flags"):
            if getattr(self, name, 0):
                _rt.cudaFree(getattr(self, name))
                setattr(self, name, 0)

    def close(self) -> None:
        """Collective over the group (every rank calls it, in the same order as the other
        exchangers' close): drain this rank's transfers, unmap the peers' buffers, and free
        this rank's own buffers once no peer maps them any more."""
        if self.closed:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # every rank's copies into its peers have landed
        self._unmap()
        dist.barrier(group=self.group)  # no peer maps this rank's buffers any more
        self._free_local()
        self.closed = True

    def next_slot(self) -> int:
        """Slots are taken round robin; every rank calls this in the same order."""
        k = self.step % self.nslots
        self.step += 1
        return k


class PeerAllToAll(_Symmetric):
    """Symmetric-buffer all-to-all among the ranks of `group` (one process per GPU, one node)."""

    def __init__(self, group, chunk_shape, dtype: torch.dtype, nslots: int = 2):
        n = dist.get_world_size(group)
        esz = torch.empty((), dtype=dtype).element_size()
        self.chunk_shape = tuple(chunk_shape)
        self.dtype = dtype
        self.chunk = int(esz * torch.Size(chunk_shape).numel())
        super().__init__(group, n * self.chunk, nslots, 2 * nslots * n)  # arrive[k][src], free[k][dst]
        self.streams = [torch.cuda.Stream() for _ in range(self.n)]
        dist.barrier(group=group)

    # flag addresses: arrive[k][src] at (k * n + src), free[k][dst] at (nslots * n + k * n + dst)
    def _arrive(self, base: int, k: int, src: int) -> int:
        return base + 4 * (k * self.n + src)

    def _free(self, base: int, k: int, dst: int) -> int:
        return base + 4 * (self.nslots * self.n + k * self.n + dst)

    def recv_tensor(self, k: int) -> torch.Tensor:
        """Slot k of this rank's receive buffer as (n, *chunk_shape): [src] = what src sent."""
        return _RawArray(self.data + k * self.slot, (self.n,) + self.chunk_shape, self.dtype).tensor()

    def send(self, send: torch.Tensor, k: int) -> int:
        """Start the transfer of send (n, *chunk_shape), [dst] to rank dst, into slot k of every
        rank: copy-engine copies on per-destination side streams after the current stream's
        work so far; the current stream does not wait for them (see wait). Returns the slot's
        use number, which wait / release take when several uses are in flight."""
        if tuple(send.shape) != (self.n,) + self.chunk_shape or send.dtype != self.dtype or not send.is_contiguous():
            raise ValueError("send must be a contiguous (n_ranks, *chunk_shape) tensor of the exchange dtype")
        cur = torch.cuda.current_stream()
        u = self.use[k] + 1
        self.use[k] = u
        src_base = send.data_ptr()
        ev = torch.cuda.Event()
        ev.record(cur)
        if not hasattr(self, "_local_done"):
            self._local_done = {}
        for d in range(self.n):
            st = self.streams[d]
            st.wait_event(ev)
            h = st.cuda_stream
            if d != self.r:  # d has consumed use u-1 of its slot k
                _ck(_cu.cuStreamWaitValue32(h, self._free(self.flags, k, d), u - 1, _GEQ))
            dst = self.peer_data[d] + k * self.slot + self.r * self.chunk
            _ck(_rt.cudaMemcpyAsync(dst, src_base + d * self.chunk, self.chunk, _D2D, h))
            if d != self.r:
                _ck(_cu.cuStreamWriteValue32(h, self._arrive(self.peer_flags[d], k, self.r), u, _WDEF))
            else:
                e = torch.cuda.Event()
                e.record(st)
                self._local_done[(k, u)] = e
            send.record_stream(st)  # the allocator keeps send alive until the copy ran
        return u

    def wait(self, k: int, u: int | None = None) -> torch.Tensor:
        """The current stream waits until every rank's chunk of use u (default: the latest) of
        slot k has landed; returns slot k of the receive buffer as (n, *chunk_shape)."""
        u = self.use[k] if u is None else u
        cur = torch.cuda.current_stream()
        cur.wait_event(self._local_done.pop((k, u)))
        h = cur.cuda_stream
        for s in range(self.n):
            if s != self.r:
                _ck(_cu.cuStreamWaitValue32(h, self._arrive(self.flags, k, s), u, _GEQ))
        return self.recv_tensor(k)

    def exchange(self, send: torch.Tensor, k: int) -> torch.Tensor:
        """send + wait: enqueued on the current stream; returns slot k of the receive buffer
        (valid on that stream)."""
        self.send(send, k)
        return self.wait(k)

    def release(self, k: int, u: int | None = None) -> None:
        """Enqueue on the current stream (after the last reader of slot k): tell every sender
        that this rank is done with use u (default: the latest) of slot k."""
        u = self.use[k] if u is None else u
        h = torch.cuda.current_stream().cuda_stream
        for s in range(self.n):
            if s != self.r:
                _ck(_cu.cuStreamWriteValue32(h, self._free(self.peer_flags[s], k, self.r), u, _WDEF))


class PeerHalo(_Symmetric):
    """Causal halo to the next rank (the p2p scheme's one message per boundary, cpsim.py:475-485)
    as one copy-engine copy into rank r+1's symmetric slot plus a fenced flag write: no NCCL
    kernel, no SMs, so the transfer hides behind the projection GEMM that follows it.

    Flags: arrive[k] (written by r-1), free[k] (written by r+1). Per-slot use counters give
    the same flow control as PeerAllToAll."""

    def __init__(self, group, shape, dtype: torch.dtype, nslots: int = 2):
        self.shape = tuple(shape)
        self.dtype = dtype
        nbytes = int(torch.empty((), dtype=dtype).element_size() * torch.Size(shape).numel())
        super().__init__(group, nbytes, nslots, 2 * nslots)
        self.side = torch.cuda.Stream()
        dist.barrier(group=group)

    def send(self, tail: torch.Tensor, k: int):
        """Enqueue (after the current stream's work) the copy of `tail` into rank r+1's slot k;
        returns slot k of this rank's buffer (rank r-1's halo; None on rank 0). Call wait(k)
        on the consuming stream before reading it."""
        if tuple(tail.shape) != self.shape or tail.dtype != self.dtype or not tail.is_contiguous():
            raise ValueError("halo must be a contiguous tensor of the exchange shape and dtype")
        u = self.use[k] + 1
        self.use[k] = u
        if self.r < self.n - 1:
            cur = torch.cuda.current_stream()
            self.side.wait_stream(cur)
            h = self.side.cuda_stream
            d = self.r + 1
            _ck(_cu.cuStreamWaitValue32(h, self.flags + 4 * (self.nslots + k), u - 1, _GEQ))
            _ck(_rt.cudaMemcpyAsync(self.peer_data[d] + k * self.slot, tail.data_ptr(), self.slot, _D2D, h))
            _ck(_cu.cuStreamWriteValue32(h, self.peer_flags[d] + 4 * k, u, _WDEF))
            tail.record_stream(self.side)
        if self.r == 0:
            return None
        if not hasattr(self, "_views"):
            self._views = [_RawArray(self.data + j * self.slot, self.shape, self.dtype).tensor()
                           for j in range(self.nslots)]
        return self._views[k]

    def wait(self, k: int) -> None:
        """Current stream waits until rank r-1's halo for slot k's current use has landed."""
        if self.r > 0:
            _ck(_cu.cuStreamWaitValue32(torch.cuda.current_stream().cuda_stream, self.flags + 4 * k,
                                        self.use[k], _GEQ))

    def release(self, k: int) -> None:
        """Enqueue after the last reader of slot k: rank r-1 may overwrite it."""
        if self.r > 0:
            _ck(_cu.cuStreamWriteValue32(torch.cuda.current_stream().cuda_stream,
                                         self.peer_flags[self.r - 1] + 4 * (self.nslots + k), self.use[k], _WDEF))
