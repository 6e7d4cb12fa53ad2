"""fp32 projections on the tensor cores by three-way bf16 splitting.

The fp32 operator path (config C1) is dominated by its projection GEMMs. Native fp32 GEMMs
run on the CUDA cores (SIMT, ~65 TFLOP/s on B200) and TF32 would break the 1e-5 parity bar.
Every fp32 value is exactly the sum of three bf16 values, x = x0 + x1 + x2 (8 + 8 + 8 mantissa
bits), so

    A @ B = sum_{i + j <= 2} Ai @ Bj  + O(2^-24 |A| |B|)

takes six bf16 tensor-core products with fp32 accumulation (the dropped terms are below fp32
rounding). The weight splits are made once per operator; the activation split is one
kernel (hy_split3_cat, csrc/split3.cu) writing the K-concatenated operand. The five small products run as ONE GEMM with the splits concatenated along
K (Split3.cat, K' = 5K); the leading term A0 @ B0 follows, accumulated into the same fp32
output (cuBLAS beta = 1). The error is set by the fp32 accumulation inside a long-K
tensor-core GEMM, so the leading term is accumulated in K chunks with fp32 adds between them.
Measured on B200 at the C1 projection (M = 12288, K = N = 4096, `scripts/split3_err.py`):
one K = 4096 pass 5.8e-6 relative to max, chunks of 2048 2.8e-6 (1.73 ms), of 1024 1.3e-6
(1.85 ms, used: the operator composes two GEMMs and three gated rows, and with 2048-chunks the
C1 / fp32-C3 operator parity measured 8.5-8.8e-6 against the 1e-5 bar); cuBLAS's CUDA-core
fp32 GEMM: 3.0e-6 at 6.27 ms.
"""

from __future__ import annotations

import torch

_PAIRS = ((1, 1), (0, 2), (2, 0), (0, 1), (1, 0))  # smallest terms first; A0 @ B0 last, K-chunked
_KC = 1024


class Split3(tuple):
    """split3 parts of a weight plus `cat` = [A1 | A0 | A2 | A0 | A1] (M, 5K): the five small
    products of _PAIRS as ONE bf16 GEMM against [B1; B2; B0; B1; B0] (K' = 5K). Their
    magnitudes are <= 2^-8 of the result, so the long-K fp32 accumulation error of that GEMM is
    negligible, and one GEMM replaces five output read-modify-write passes."""

    cat: torch.Tensor


def split3_weight(a: torch.Tensor) -> Split3:
    parts = Split3(split3(a))
    parts.cat = torch.cat([parts[i] for i, _ in _PAIRS], dim=1).contiguous()
    return parts


def _b_cat(b_parts) -> torch.Tensor:
    if isinstance(b_parts, Split3Act):
        return b_parts.cat
    return torch.cat([b_parts[j] for _, j in _PAIRS], dim=-2)


class Split3Act:
    """An activation's split in the K-concatenated operand layout, made by one kernel
    (hy_split3_cat): cat = [X1; X2; X0; X1; X0] ((Bt,) 5K, N) bf16, the B operand of the five
    small products (the order of _PAIRS); its last K rows are X0, the leading product's."""

    def __init__(self, cat: torch.Tensor, K: int):
        self.cat = cat
        self.K = K

    def __getitem__(self, j: int) -> torch.Tensor:
        if j != 0:
            raise IndexError("Split3Act exposes only the leading part X0 (index 0) and .cat")
        return self.cat[..., 4 * self.K:, :]

    def batch(self, i: int) -> "Split3Act":
        return Split3Act(self.cat[i], self.K)


def split3_act(x: torch.Tensor) -> Split3Act:
    """fp32 (K, N) or (Bt, K, N) CUDA activation -> Split3Act in one HBM pass (hy_split3_cat)."""
    from . import _lib
    if x.dtype != torch.float32 or not x.is_cuda:
        raise ValueError("split3_act takes a float32 CUDA tensor")
    x = x.contiguous()
    x3 = x.unsqueeze(0) if x.dim() == 2 else x
    Bt, K, N = x3.shape
    cat = torch.empty((Bt, 5 * K, N), dtype=torch.bfloat16, device=x.device)
    lib = _lib.load()
    _lib.check(lib.hy_split3_cat(x3.data_ptr(), cat.data_ptr(), Bt, K, N,
                                 torch.cuda.current_stream().cuda_stream), "split3_cat")
    return Split3Act(cat[0] if x.dim() == 2 else cat, K)


def split3(a: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """fp32 a -> (a0, a1, a2) bf16 with a0 + a1 + a2 == a (to fp32 precision)."""
    a0 = a.to(torch.bfloat16)
    r = a - a0.float()
    a1 = r.to(torch.bfloat16)
    a2 = (r - a1.float()).to(torch.bfloat16)
    return a0, a1, a2


def matmul_split3(a_parts, b_parts, out: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    """fp32 A @ B from split3 parts: A (M, K), B (K, N) or batched (Bt, K, N) with shared A.
    accumulate: out += A @ B (out must be given)."""
    a0 = a_parts[0]
    b0 = b_parts[0]
    if accumulate and out is None:
        raise ValueError("accumulate needs out")
    if b0.dim() == 3:
        Bt, _, N = b0.shape
        if out is None:
            out = torch.empty((Bt, a0.shape[0], N), dtype=torch.float32, device=a0.device)
        for i in range(Bt):
            bi = b_parts.batch(i) if isinstance(b_parts, Split3Act) else tuple(p[i] for p in b_parts)
            matmul_split3(a_parts, bi, out=out[i], accumulate=accumulate)
        return out
    if out is None:
        out = torch.empty((a0.shape[0], b0.shape[1]), dtype=torch.float32, device=a0.device)
    cat = getattr(a_parts, "cat", None)
    if cat is not None:  # the five small products in one GEMM
        bc = _b_cat(b_parts)
        if accumulate:
            torch.addmm(out, cat, bc, out_dtype=torch.float32, out=out)
        else:
            torch.mm(cat, bc, out_dtype=torch.float32, out=out)
    else:
        if isinstance(b_parts, Split3Act):
            raise ValueError("a Split3Act operand needs a weight split made by split3_weight")
        first = not accumulate
        for i, j in _PAIRS:
            if first:
                torch.mm(a_parts[i], b_parts[j], out_dtype=torch.float32, out=out)
                first = False
            else:
                torch.addmm(out, a_parts[i], b_parts[j], out_dtype=torch.float32, out=out)
    K = a0.shape[1]
    for k0 in range(0, K, _KC):
        torch.addmm(out, a0[:, k0:k0 + _KC], b0[k0:k0 + _KC], out_dtype=torch.float32, out=out)
    return out
