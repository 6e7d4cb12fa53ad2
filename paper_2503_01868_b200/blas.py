"""fp32 projections on the tensor cores by three-way bf16 splitting.

The fp32 operator path (config C1) is dominated by its projection GEMMs. Native fp32 GEMMs
run on the CUDA cores (SIMT, ~65 TFLOP/s on B200) and TF32 would break the 1e-5 parity bar.
Every fp32 value is exactly the sum of three bf16 values, x = x0 + x1 + x2 (8 + 8 + 8 mantissa
bits), so

    A @ B = sum_{i + j <= 2} Ai @ Bj  + O(2^-24 |A| |B|)

takes six bf16 tensor-core GEMMs with fp32 accumulation (the dropped terms are below fp32
rounding). The weight splits are made once per operator; the activation split is one
elementwise pass. Products are accumulated smallest first into one fp32 output (cuBLAS
beta = 1). Measured on B200 at the C1 projection (M = 12288, K = N = 4096): the error is set by
the fp32 accumulation inside a long-K tensor-core GEMM (5.0e-6 relative to max with one
K = 4096 pass), so the leading term A0 @ B0 is accumulated in K chunks of 1024 with fp32 adds
between them: 1.2e-6, against 3.0e-6 for cuBLAS's CUDA-core fp32 GEMM, at 3.2x its speed
(1.99 ms vs 6.27 ms).
"""

from __future__ import annotations

import torch

_PAIRS = ((1, 1), (0, 2), (2, 0), (0, 1), (1, 0))  # smallest terms first; A0 @ B0 last, K-chunked
_KC = 1024


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
            matmul_split3(a_parts, tuple(p[i] for p in b_parts), out=out[i], accumulate=accumulate)
        return out
    if out is None:
        out = torch.empty((a0.shape[0], b0.shape[1]), dtype=torch.float32, device=a0.device)
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
