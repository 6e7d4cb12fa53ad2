"""Torch-native device entry points over the C-ABI (no host copies, no fallback).

Every function takes CUDA tensors in the (B, C, L) layout (a 2-D (C, L) tensor
is treated as B = 1), launches one of the sm_100a kernels on the current torch
stream and returns a new CUDA tensor. Filter taps are per group, (G, lh),
float32 for fp32/bf16 activations and float64 for fp64 ones.
"""

from __future__ import annotations

import torch

from . import _lib

_DT = {torch.float32: _lib.HY_F32, torch.bfloat16: _lib.HY_BF16, torch.float64: _lib.HY_F64}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _as3(x: torch.Tensor) -> torch.Tensor:
    if x.dim() == 2:
        return x.unsqueeze(0)
    if x.dim() != 3:
        raise ValueError(f"expected (B, C, L) or (C, L), got shape {tuple(x.shape)}")
    return x


def _check_device(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("paper_2503_01868_b200 ops need CUDA tensors (there is no CPU path)")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")


def _dtype_code(x: torch.Tensor) -> int:
    try:
        return _DT[x.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {x.dtype}; use float32, bfloat16 or float64") from None


def tap_dtype(act_dtype: torch.dtype) -> torch.dtype:
    return torch.float64 if act_dtype == torch.float64 else torch.float32


def _taps(taps: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    want = tap_dtype(x.dtype)
    if taps.dtype != want or not taps.is_contiguous() or taps.device != x.device:
        taps = taps.to(device=x.device, dtype=want).contiguous()
    return taps


def causal_conv(x: torch.Tensor, taps: torch.Tensor, group_size: int = 1) -> torch.Tensor:
    """y = h conv x per channel (core.py:212-226), any filter length. x: (B,C,L) or (C,L)."""
    squeeze = x.dim() == 2
    x3 = _as3(x)
    _check_device(x3)
    taps = _taps(taps, x3)
    B, C, L = x3.shape
    lh = taps.shape[-1]
    y = torch.empty_like(x3)
    lib = _lib.load()
    _lib.check(lib.hy_causal_conv_fwd(x3.data_ptr(), y.data_ptr(), taps.data_ptr(), B, C, L, lh,
                                      group_size, _dtype_code(x3), _stream()), "causal_conv")
    return y[0] if squeeze else y


def gated_conv(v: torch.Tensor, taps: torch.Tensor, group_size: int = 1, q=None, k=None) -> torch.Tensor:
    """y = q * conv(k * v) on CUDA cores (blockconv.py:182-220 semantics, any lh)."""
    squeeze = v.dim() == 2
    v3, q3, k3 = _as3(v), None if q is None else _as3(q), None if k is None else _as3(k)
    _check_device(v3, q3, k3)
    for name, g in (("q", q3), ("k", k3)):
        if g is not None and (g.shape != v3.shape or g.dtype != v3.dtype):
            raise ValueError(f"gate {name} shape/dtype {tuple(g.shape)}/{g.dtype} does not match input "
                             f"{tuple(v3.shape)}/{v3.dtype}")
    taps = _taps(taps, v3)
    B, C, L = v3.shape
    y = torch.empty_like(v3)
    lib = _lib.load()
    _lib.check(lib.hy_gated_conv_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), taps.data_ptr(), B, C,
                                     L, taps.shape[-1], group_size, _dtype_code(v3), _stream()),
               "gated_conv")
    return y[0] if squeeze else y


def two_stage(v: torch.Tensor, taps_hat: torch.Tensor, group_size: int = 1, q=None, k=None,
              decay=None) -> torch.Tensor:
    """tcgen05 two-stage conv, bf16 (blockconv.py:160-220): y = q * (T0 U_n + T1 U_{n-1}).

    taps_hat: (G, lh) fp32 with lh <= 129; decay: (G,) fp32 = rate*log2(base) or None.
    """
    squeeze = v.dim() == 2
    v3, q3, k3 = _as3(v), None if q is None else _as3(q), None if k is None else _as3(k)
    _check_device(v3, q3, k3)
    if v3.dtype != torch.bfloat16:
        raise ValueError("two_stage (tcgen05) takes bfloat16 activations; use gated_conv for fp32/fp64")
    for name, g in (("q", q3), ("k", k3)):
        if g is not None and (g.shape != v3.shape or g.dtype != v3.dtype):
            raise ValueError(f"gate {name} shape {tuple(g.shape)} does not match input {tuple(v3.shape)}")
    taps_hat = taps_hat.to(device=v3.device, dtype=torch.float32).contiguous()
    if decay is not None:
        decay = decay.to(device=v3.device, dtype=torch.float32).contiguous()
    B, C, L = v3.shape
    y = torch.empty_like(v3)
    lib = _lib.load()
    _lib.check(lib.hy_two_stage_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), taps_hat.data_ptr(),
                                    _ptr(decay), B, C, L, taps_hat.shape[-1], group_size, _lib.HY_BF16,
                                    _stream()), "two_stage")
    return y[0] if squeeze else y


BLOCK_CONV_MAX_LH = 513  # hy_block_conv_fwd: K <= 4 spill factors of 128


def block_conv(v: torch.Tensor, taps_hat: torch.Tensor, group_size: int = 1, q=None, k=None,
               decay=None) -> torch.Tensor:
    """tcgen05 K-block conv, bf16 (blockconv.py:103-121, gated as blockconv.py:182-220):
    y = q * sum_k T_k U_{n-k}, any filter length up to 513 taps.

    taps_hat: (G, lh) fp32; decay: (G,) fp32 = rate*log2(base) or None."""
    squeeze = v.dim() == 2
    v3, q3, k3 = _as3(v), None if q is None else _as3(q), None if k is None else _as3(k)
    _check_device(v3, q3, k3)
    if v3.dtype != torch.bfloat16:
        raise ValueError("block_conv (tcgen05) takes bfloat16 activations; use causal_conv for fp32/fp64")
    for name, g in (("q", q3), ("k", k3)):
        if g is not None and (g.shape != v3.shape or g.dtype != v3.dtype):
            raise ValueError(f"gate {name} shape {tuple(g.shape)} does not match input {tuple(v3.shape)}")
    taps_hat = taps_hat.to(device=v3.device, dtype=torch.float32).contiguous()
    if decay is not None:
        decay = decay.to(device=v3.device, dtype=torch.float32).contiguous()
    B, C, L = v3.shape
    if L % 8:  # the kernel streams 16-byte row pieces; zero steps after L change no output <= L
        pad = lambda t: None if t is None else torch.nn.functional.pad(t, (0, 8 - L % 8)).contiguous()  # noqa: E731
        y = block_conv(pad(v3), taps_hat, group_size, q=pad(q3), k=pad(k3), decay=decay)[..., :L].contiguous()
        return y[0] if squeeze else y
    y = torch.empty_like(v3)
    lib = _lib.load()
    _lib.check(lib.hy_block_conv_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), taps_hat.data_ptr(),
                                     _ptr(decay), B, C, L, taps_hat.shape[-1], group_size, _lib.HY_BF16,
                                     _stream()), "block_conv")
    return y[0] if squeeze else y


def feat_pack(feat_taps: torch.Tensor) -> torch.Tensor:
    """Pack (3, C, lhf) featurizer taps for the tcgen05 mixer (hy_feat_pack)."""
    ft = feat_taps.to(dtype=torch.float32).contiguous()
    _check_device(ft)
    _, C, lhf = ft.shape
    lib = _lib.load()
    out = torch.empty(int(lib.hy_feat_pack_size(C, lhf)), dtype=torch.uint8, device=ft.device)
    _lib.check(lib.hy_feat_pack(ft.data_ptr(), C, lhf, out.data_ptr(), _stream()), "feat_pack")
    return out


def hyena_mixer(proj: torch.Tensor, feat_taps: torch.Tensor, inner_taps: torch.Tensor, group_size: int,
                decay=None, out=None, se_only: bool = False, packed=None, hist=None) -> torch.Tensor:
    """Fused featurizers + gates + inner conv (hyena.py:162-186) from the (B, 3C, L) projections.

    feat_taps: (3, C, lhf) per-channel [q, k, v] featurizer taps (fp32);
    inner_taps: (G, lh) fp32; decay: (G,) fp32 or None;
    hist: (B, 3C, 144) projections before t = 0 (context parallel), None = zeros.
    """
    _check_device(proj)
    B, C3, L = proj.shape
    if C3 % 3 != 0:
        raise ValueError("proj must be (B, 3C, L)")
    C = C3 // 3
    ft = feat_taps.to(device=proj.device, dtype=torch.float32).contiguous()
    it = inner_taps.to(device=proj.device, dtype=torch.float32).contiguous()
    if decay is not None:
        decay = decay.to(device=proj.device, dtype=torch.float32).contiguous()
    if ft.shape[:2] != (3, C):
        raise ValueError(f"feat_taps must be (3, {C}, lhf), got {tuple(ft.shape)}")
    y = out if out is not None else torch.empty((B, C, L), device=proj.device, dtype=proj.dtype)
    lib = _lib.load()
    if se_only:
        _lib.check(lib.hy_se_mixer_fwd(proj.data_ptr(), y.data_ptr(), ft.data_ptr(), ft.shape[-1], it.data_ptr(),
                                       _ptr(decay), it.shape[-1], group_size, B, C, L, _dtype_code(proj),
                                       _stream()), "se_mixer")
        return y
    if packed is None and proj.dtype == torch.bfloat16:
        packed = feat_pack(ft)
    if hist is not None:
        _check_device(hist)
        if tuple(hist.shape) != (B, C3, _lib.MIXER_HISTORY) or hist.dtype != proj.dtype:
            raise ValueError(f"hist must be (B, 3C, {_lib.MIXER_HISTORY}) {proj.dtype}")
    _lib.check(lib.hy_hyena_mixer_fwd(proj.data_ptr(), y.data_ptr(), ft.data_ptr(), _ptr(packed), _ptr(hist),
                                      ft.shape[-1],
                                      it.data_ptr(), _ptr(decay), it.shape[-1], group_size, B, C, L,
                                      _dtype_code(proj), _stream()), "hyena_mixer")
    return y


def halo_correction(halo: torch.Tensor, y: torch.Tensor, taps: torch.Tensor, group_size: int = 1) -> None:
    """In place: y[..., t] += sum_{j>t} h[j] halo[..., H+t-j] for t < H (cpsim.py:498-510)."""
    h3, y3 = _as3(halo), _as3(y)
    _check_device(h3, y3)
    taps = _taps(taps, y3)
    B, C, L = y3.shape
    lib = _lib.load()
    _lib.check(lib.hy_halo_correction_fwd(h3.data_ptr(), y3.data_ptr(), taps.data_ptr(), B, C, L,
                                          taps.shape[-1], group_size, _dtype_code(y3), _stream()),
               "halo_correction")


class FFTSpectrum:
    """Cached spectra of a filter bank's zero-padded taps (hy_fft_spectrum): `data` is a
    (G, N, 2) float32 device tensor in the register four-step path's own order, valid for
    sequence length L and filter length lh."""

    def __init__(self, data: torch.Tensor, L: int, lh: int):
        self.data, self.L, self.lh = data, L, lh


def fft_spectrum(taps: torch.Tensor, L: int):
    """Spectra of (G, lh) taps for sequences of length L, or None where the cached path does not
    cover N = next_pow2(L + lh - 1) (2^14 <= N <= 2^18)."""
    if not taps.is_cuda:
        raise ValueError("paper_2503_01868_b200 ops need CUDA tensors (there is no CPU path)")
    taps = taps.to(torch.float32).contiguous()
    G, lh = taps.shape
    lib = _lib.load()
    nbytes = int(lib.hy_fft_spectrum_size(G, L, lh))
    if nbytes == 0:
        return None
    spec = torch.empty((nbytes // 4,), dtype=torch.float32, device=taps.device).view(G, -1, 2)
    ws_bytes = int(lib.hy_fft_conv_workspace_size(1, G, L, lh, 1, _lib.HY_F32))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=taps.device)
    _lib.check(lib.hy_fft_spectrum(taps.data_ptr(), G, L, lh, spec.data_ptr(), ws.data_ptr(), ws_bytes, _stream()),
               "fft_spectrum")
    return FFTSpectrum(spec, L, lh)


def fft_conv(v: torch.Tensor, taps: torch.Tensor, group_size: int = 1, q=None, k=None,
             spectrum: FFTSpectrum | None = None) -> torch.Tensor:
    """y = q * (h conv (k * v)) through the FFT kernel (fft.py:128-145, hyena.py:183-186);
    `spectrum` (from fft_spectrum(taps, L)) skips the filter transform."""
    squeeze = v.dim() == 2
    v3, q3, k3 = _as3(v), None if q is None else _as3(q), None if k is None else _as3(k)
    _check_device(v3, q3, k3)
    B, C, L = v3.shape
    lib = _lib.load()
    code = _dtype_code(v3)
    y = torch.empty_like(v3)
    if spectrum is not None:
        if spectrum.L != L:
            raise ValueError(f"spectrum computed for L={spectrum.L}, input has L={L}")
        lh = spectrum.lh
        ws_bytes = lib.hy_fft_conv_workspace_size(B, C, L, lh, group_size, code)
        ws = torch.empty(max(int(ws_bytes), 1), dtype=torch.uint8, device=v3.device)
        _lib.check(lib.hy_fft_conv_spec_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), spectrum.data.data_ptr(),
                                            B, C, L, lh, group_size, code, ws.data_ptr(), int(ws_bytes), _stream()),
                   "fft_conv")
        return y[0] if squeeze else y
    taps = _taps(taps, v3)
    lh = taps.shape[-1]
    ws_bytes = lib.hy_fft_conv_workspace_size(B, C, L, lh, group_size, code)
    ws = torch.empty(max(int(ws_bytes), 1), dtype=torch.uint8, device=v3.device)
    _lib.check(lib.hy_fft_conv_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), taps.data_ptr(), B, C, L,
                                   lh, group_size, code, ws.data_ptr(), int(ws_bytes), _stream()), "fft_conv")
    return y[0] if squeeze else y


def long_conv(v: torch.Tensor, taps: torch.Tensor, group_size: int = 1, q=None, k=None,
              spectrum: FFTSpectrum | None = None) -> torch.Tensor:
    """Gated causal conv for long filters: the FFT kernel where it covers the case, else the FIR kernel."""
    if spectrum is None and taps.shape[-1] > v.shape[-1]:
        taps = taps[..., : v.shape[-1]].contiguous()  # lags >= L never reach the L outputs
    try:
        return fft_conv(v, taps, group_size, q=q, k=k, spectrum=spectrum)
    except NotImplementedError:
        return gated_conv(v, taps, group_size, q=q, k=k)


def fft_c2c(x: torch.Tensor, inverse: bool = False) -> torch.Tensor:
    """Complex FFT of the last axis (power-of-two length, natural order) by the hand-written
    Stockham kernel (hy_fft_c2c): forward unnormalised, inverse carrying 1/n (fft.py:116-125).
    complex64 / complex128 CUDA tensors."""
    if not x.is_cuda:
        raise ValueError("paper_2503_01868_b200 ops need CUDA tensors (there is no CPU path)")
    if x.dtype not in (torch.complex64, torch.complex128):
        raise ValueError(f"fft_c2c takes complex64 / complex128, got {x.dtype}")
    n = x.shape[-1]
    xc = x.contiguous()
    batch = xc.numel() // max(n, 1)
    y = torch.empty_like(xc)
    code = _lib.HY_F64 if x.dtype == torch.complex128 else _lib.HY_F32
    lib = _lib.load()
    nbytes = int(lib.hy_fft_c2c_workspace_size(batch, n, code))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=x.device)
    _lib.check(lib.hy_fft_c2c(xc.data_ptr(), y.data_ptr(), batch, n, int(inverse), code, ws.data_ptr(), nbytes,
                              _stream()), "fft_c2c")
    return y / n if inverse else y


def gate_mul(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = a * b (hy_gate_mul): contiguous CUDA tensors of one dtype and element count."""
    _check_device(a, b, out)
    if a.numel() != b.numel() or a.dtype != b.dtype or (out is not None and (out.numel() != a.numel()
                                                                             or out.dtype != a.dtype)):
        raise ValueError("gate_mul operands must match in size and dtype")
    out = torch.empty_like(a) if out is None else out
    lib = _lib.load()
    _lib.check(lib.hy_gate_mul(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(), _dtype_code(a), _stream()),
               "gate_mul")
    return out


def qkv_weight_permute(w_qkv_t: torch.Tensor) -> torch.Tensor:
    """Row order of hy_qkv_feat_gemm's weight: the (3D, D) [W_q; W_k; W_v]^T rows regrouped as
    D/128 tiles of 128 q rows, then D/64 tiles of [64 k rows; the same channels' 64 v rows]."""
    D = w_qkv_t.shape[1]
    if w_qkv_t.shape[0] != 3 * D or D % 128:
        raise ValueError("w_qkv_t must be (3D, D) with D % 128 == 0")
    kv = torch.stack([w_qkv_t[D:2 * D].reshape(D // 64, 64, D), w_qkv_t[2 * D:].reshape(D // 64, 64, D)], dim=1)
    return torch.cat([w_qkv_t[:D], kv.reshape(2 * D, D)]).contiguous()


def qkv_feat_gemm(x: torch.Tensor, w_perm: torch.Tensor, feat_taps: torch.Tensor, segments: int = 0):
    """(fq, u), each (B, D, L): the featurizers of W_qkv^T x with u = fk * fv, in one tcgen05 GEMM
    whose epilogue runs the FIRs (hyena.py:122-126, 184). bf16,
    D % 128 == 0, L % 256 == 0, featurizers <= 8 taps; w_perm from qkv_weight_permute;
    segments = time segments per 128-row tile (0: chosen for the grid)."""
    _check_device(x, w_perm)
    x3 = _as3(x)
    B, D, L = x3.shape
    if x3.dtype != torch.bfloat16 or w_perm.dtype != torch.bfloat16:
        raise ValueError("qkv_feat_gemm takes bfloat16 activations and weights")
    if tuple(w_perm.shape) != (3 * D, D):
        raise ValueError(f"w_perm must be (3D, D) = ({3 * D}, {D})")
    if feat_taps.dim() != 3 or tuple(feat_taps.shape[:2]) != (3, D):
        raise ValueError("feat_taps must be (3, D, lhf)")
    taps = feat_taps.to(device=x3.device, dtype=torch.float32).contiguous()
    fq = torch.empty_like(x3)
    u = torch.empty_like(x3)
    lib = _lib.load()
    _lib.check(lib.hy_qkv_feat_gemm(w_perm.data_ptr(), x3.data_ptr(), taps.data_ptr(), taps.shape[2], fq.data_ptr(),
                                    u.data_ptr(), B, D, L, segments, _dtype_code(x3), _stream()), "qkv_feat_gemm")
    if x.dim() == 2:
        return fq[0], u[0]
    return fq, u


def _modes(residues: torch.Tensor, poles: torch.Tensor, dev):
    r = residues.to(device=dev, dtype=torch.float32).contiguous()
    p = poles.to(device=dev, dtype=torch.float32).contiguous()
    if r.shape != p.shape or r.dim() != 2:
        raise ValueError("residues and poles must be matching (n_groups, n_poles) tensors")
    return r, p


def li_conv(v: torch.Tensor, residues: torch.Tensor, poles: torch.Tensor, group_size: int = 1, q=None,
            k=None) -> torch.Tensor:
    """y = q * (h conv (k * v)) with h_t = sum_n R_n lam_n^t over the whole sequence (tcgen05, bf16)."""
    squeeze = v.dim() == 2
    v3, q3, k3 = _as3(v), None if q is None else _as3(q), None if k is None else _as3(k)
    _check_device(v3, q3, k3)
    if v3.dtype != torch.bfloat16:
        raise ValueError("li_conv (tcgen05) takes bfloat16 activations")
    r, p = _modes(residues, poles, v3.device)
    B, C, L = v3.shape
    y = torch.empty_like(v3)
    lib = _lib.load()
    _lib.check(lib.hy_li_conv_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), r.data_ptr(), p.data_ptr(),
                                  p.shape[1], group_size, B, C, L, _lib.HY_BF16, _stream()), "li_conv")
    return y[0] if squeeze else y


def li_scan(v: torch.Tensor, residues: torch.Tensor, poles: torch.Tensor, group_size: int = 1, q=None,
            k=None) -> torch.Tensor:
    """y = q * (h conv (k * v)), h_t = sum_n R_n lam_n^t, by exact per-mode state scans on CUDA
    cores (hy_li_scan_fwd): fp32 / bf16 / fp64 activations, up to 64 poles, any L.
    residues, poles: (n_groups, n_poles), kept in fp64."""
    squeeze = v.dim() == 2
    v3, q3, k3 = _as3(v), None if q is None else _as3(q), None if k is None else _as3(k)
    _check_device(v3, q3, k3)
    for name, gt in (("q", q3), ("k", k3)):
        if gt is not None and (gt.shape != v3.shape or gt.dtype != v3.dtype):
            raise ValueError(f"gate {name} shape/dtype {tuple(gt.shape)}/{gt.dtype} does not match input "
                             f"{tuple(v3.shape)}/{v3.dtype}")
    r = residues.to(device=v3.device, dtype=torch.float64).contiguous()
    p = poles.to(device=v3.device, dtype=torch.float64).contiguous()
    if r.shape != p.shape or r.dim() != 2:
        raise ValueError("residues and poles must be matching (n_groups, n_poles) tensors")
    B, C, L = v3.shape
    if r.shape[0] * group_size != C:
        raise ValueError(f"{r.shape[0]} filter groups of size {group_size} do not cover {C} channels")
    y = torch.empty_like(v3)
    lib = _lib.load()
    _lib.check(lib.hy_li_scan_fwd(_ptr(q3), _ptr(k3), v3.data_ptr(), y.data_ptr(), r.data_ptr(), p.data_ptr(),
                                  p.shape[1], group_size, B, C, L, _dtype_code(v3), _stream()), "li_scan")
    return y[0] if squeeze else y


def li_scan_mixer(proj: torch.Tensor, feat_taps: torch.Tensor, residues: torch.Tensor, poles: torch.Tensor,
                  group_size: int = 1) -> torch.Tensor:
    """LI mixer on the modal scan (hy_li_scan_mixer_fwd): featurizers (lhf <= 8) + gates + the
    implicit long conv from the (B, 3C, L) projections in one pass; fp32 / bf16 / fp64."""
    _check_device(proj)
    B, C3, L = proj.shape
    if C3 % 3:
        raise ValueError("proj must be (B, 3C, L)")
    C = C3 // 3
    ft = feat_taps.to(device=proj.device, dtype=tap_dtype(proj.dtype)).contiguous()
    if ft.shape[:2] != (3, C):
        raise ValueError(f"feat_taps must be (3, {C}, lhf), got {tuple(ft.shape)}")
    r = residues.to(device=proj.device, dtype=torch.float64).contiguous()
    p = poles.to(device=proj.device, dtype=torch.float64).contiguous()
    if r.shape != p.shape or r.dim() != 2 or r.shape[0] * group_size != C:
        raise ValueError("residues / poles must be matching (n_groups, n_poles) tensors covering the channels")
    y = torch.empty((B, C, L), device=proj.device, dtype=proj.dtype)
    lib = _lib.load()
    _lib.check(lib.hy_li_scan_mixer_fwd(proj.data_ptr(), y.data_ptr(), ft.data_ptr(), ft.shape[-1], r.data_ptr(),
                                        p.data_ptr(), p.shape[1], group_size, B, C, L, _dtype_code(proj),
                                        _stream()), "li_scan_mixer")
    return y


def li_conv_segmented(buf: torch.Tensor, residues: torch.Tensor, poles: torch.Tensor, group_size: int = 1,
                      out=None) -> torch.Tensor:
    """Ungated implicit long conv of a (n_seg, C, seg_len) buffer whose row c is the time
    concatenation of buf[0, c], buf[1, c], ... (the rank-major all-to-all buffer of the
    context-parallel LI layer); returns y in the same layout (tcgen05, bf16)."""
    if buf.dim() != 3:
        raise ValueError("segmented buffer must be (n_seg, C, seg_len)")
    _check_device(buf)
    if buf.dtype != torch.bfloat16:
        raise ValueError("li_conv (tcgen05) takes bfloat16 activations")
    buf = buf.contiguous()
    n, C, m = buf.shape
    r, p = _modes(residues, poles, buf.device)
    y = torch.empty_like(buf) if out is None else out
    lib = _lib.load()
    _lib.check(lib.hy_li_conv_segmented_fwd(buf.data_ptr(), y.data_ptr(), r.data_ptr(), p.data_ptr(), p.shape[1],
                                            group_size, C, n * m, m, C * m, _lib.HY_BF16, _stream()),
               "li_conv_segmented")
    return y


def li_mixer(proj: torch.Tensor, feat_taps: torch.Tensor, residues: torch.Tensor, poles: torch.Tensor,
             group_size: int, packed=None) -> torch.Tensor:
    """Hyena-LI mixer from the (B, 3C, L) projections: featurizers, gates, implicit long conv."""
    _check_device(proj)
    B, C3, L = proj.shape
    C = C3 // 3
    ft = feat_taps.to(device=proj.device, dtype=torch.float32).contiguous()
    if packed is None:
        packed = feat_pack(ft)
    r, p = _modes(residues, poles, proj.device)
    y = torch.empty((B, C, L), device=proj.device, dtype=proj.dtype)
    lib = _lib.load()
    _lib.check(lib.hy_li_mixer_fwd(proj.data_ptr(), y.data_ptr(), ft.data_ptr(), packed.data_ptr(), ft.shape[-1],
                                   r.data_ptr(), p.data_ptr(), p.shape[1], group_size, B, C, L,
                                   _dtype_code(proj), _stream()), "li_mixer")
    return y


# ---------------------------------------------------------------- backward


def causal_conv_bwd(dy: torch.Tensor, x, taps, group_size: int = 1, want_dx: bool = True,
                    want_dtaps: bool = True):
    """Adjoints of y = h conv x (core.py:245-268): (dx, dtaps) with
    dx[t] = sum_j h[j] dy[t+j] and dtaps[g, j] = sum_{c in g, b, t} dy[t] x[t-j].

    dy, x: (B, C, L) or (C, L); taps: (G, lh). Either output may be skipped (None returned);
    dtaps needs x and its length is taps.shape[-1] (or pass taps=None with want_dx=False and
    an int lh via `taps`)."""
    squeeze = dy.dim() == 2
    dy3 = _as3(dy)
    x3 = None if x is None else _as3(x)
    _check_device(dy3, x3)
    if x3 is not None and (x3.shape != dy3.shape or x3.dtype != dy3.dtype):
        raise ValueError(f"x {tuple(x3.shape)}/{x3.dtype} does not match dy {tuple(dy3.shape)}/{dy3.dtype}")
    B, C, L = dy3.shape
    if isinstance(taps, int):
        lh, tp = taps, None
        if want_dx:
            raise ValueError("dx needs the taps tensor")
    else:
        tp = _taps(taps, dy3)
        lh = tp.shape[-1]
    if C % group_size != 0:
        raise ValueError(f"group_size {group_size} does not divide channel count {C}")
    code = _dtype_code(dy3)
    lib = _lib.load()
    dx = torch.empty_like(dy3) if want_dx else None
    dtaps = ws = None
    if want_dtaps:
        if x3 is None:
            raise ValueError("dtaps needs x")
        dtaps = torch.empty((C // group_size, lh), dtype=tap_dtype(dy3.dtype), device=dy3.device)
        nbytes = int(lib.hy_causal_conv_bwd_workspace_size(B, C, L, lh, code))
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dy3.device)
    _lib.check(lib.hy_causal_conv_bwd(dy3.data_ptr(), _ptr(x3), _ptr(dx), _ptr(dtaps), _ptr(tp), B, C, L, lh,
                                      group_size, code, _ptr(ws), 0 if ws is None else ws.numel(), _stream()),
               "causal_conv_bwd")
    if dx is not None and squeeze:
        dx = dx[0]
    return dx, dtaps


def li_param_grad(dc: torch.Tensor, u: torch.Tensor, residues: torch.Tensor, poles: torch.Tensor,
                  group_size: int = 1):
    """(d_residues, d_poles), each (G, n_poles) fp32, of sum(dc * (h conv u)) for the implicit
    filter h_t = sum_n R_n lam_n^t — filter_param_grads(ImplicitFilter, causal_conv_taps_grad(dc, u))
    (hyena.py:193-211, core.py:255-268) by exact per-mode scans, no length-L tap gradient."""
    dc3, u3 = _as3(dc), _as3(u)
    _check_device(dc3, u3)
    if dc3.shape != u3.shape or dc3.dtype != u3.dtype:
        raise ValueError("dc and u must match in shape and dtype")
    r, p = _modes(residues, poles, dc3.device)
    B, C, L = dc3.shape
    if L % 8:  # the kernel streams 16-byte rows; zero steps after L contribute nothing
        pad = 8 - L % 8
        dc3 = torch.nn.functional.pad(dc3, (0, pad)).contiguous()
        u3 = torch.nn.functional.pad(u3, (0, pad)).contiguous()
        L += pad
    lib = _lib.load()
    d_res = torch.empty_like(r)
    d_pole = torch.empty_like(p)
    ws = torch.empty(int(lib.hy_li_param_grad_workspace_size(B, C)), dtype=torch.uint8, device=dc3.device)
    _lib.check(lib.hy_li_param_grad(dc3.data_ptr(), u3.data_ptr(), r.data_ptr(), p.data_ptr(), p.shape[1],
                                    group_size, B, C, L, _dtype_code(dc3), d_res.data_ptr(), d_pole.data_ptr(),
                                    ws.data_ptr(), ws.numel(), _stream()), "li_param_grad")
    return d_res, d_pole


def featurizer_bwd(proj: torch.Tensor, dmixed: torch.Tensor, conv_out: torch.Tensor, du: torch.Tensor,
                   feat_taps: torch.Tensor, du_reversed: bool = False):
    """Fused featurizer backward (hy_featurizer_bwd): (dproj (B, 3C, L), dfeat (3, C, lhf) fp32)
    from the projections, the mixer-output gradient, the inner conv output and du (stored
    time-reversed per row when du_reversed)."""
    _check_device(proj, dmixed, conv_out, du)
    B, C3, L = proj.shape
    C = C3 // 3
    for name, t in (("dmixed", dmixed), ("conv_out", conv_out), ("du", du)):
        if tuple(t.shape) != (B, C, L) or t.dtype != proj.dtype:
            raise ValueError(f"{name} must be ({B}, {C}, {L}) {proj.dtype}, got {tuple(t.shape)} {t.dtype}")
    ft = feat_taps.to(device=proj.device, dtype=torch.float32).contiguous()
    lhf = ft.shape[-1]
    lib = _lib.load()
    dproj = torch.empty_like(proj)
    dfeat = torch.empty((3, C, lhf), dtype=torch.float32, device=proj.device)
    ws = torch.empty(int(lib.hy_featurizer_bwd_workspace_size(C, lhf)), dtype=torch.uint8, device=proj.device)
    _lib.check(lib.hy_featurizer_bwd(proj.data_ptr(), dmixed.data_ptr(), conv_out.data_ptr(), du.data_ptr(),
                                     ft.data_ptr(), lhf, B, C, L, _dtype_code(proj), dproj.data_ptr(),
                                     dfeat.data_ptr(), ws.data_ptr(), ws.numel(), int(du_reversed), _stream()),
               "featurizer_bwd")
    return dproj, dfeat


def mixer_bwd_prep(proj: torch.Tensor, dmixed: torch.Tensor, feat_taps: torch.Tensor, reversed_dc: bool = False):
    """(u, dc[, dc_rev]) = ((Fk conv pk) * (Fv conv pv), dmixed * (Fq conv pq)[, dc time-reversed])
    in one stream (hy_mixer_bwd_prep)."""
    _check_device(proj, dmixed)
    B, C3, L = proj.shape
    C = C3 // 3
    if tuple(dmixed.shape) != (B, C, L) or dmixed.dtype != proj.dtype:
        raise ValueError("dmixed must be (B, C, L) of the projections' dtype")
    ft = feat_taps.to(device=proj.device, dtype=torch.float32).contiguous()
    u = torch.empty_like(dmixed)
    dc = torch.empty_like(dmixed)
    dc_rev = torch.empty_like(dmixed) if reversed_dc else None
    lib = _lib.load()
    _lib.check(lib.hy_mixer_bwd_prep(proj.data_ptr(), dmixed.data_ptr(), ft.data_ptr(), ft.shape[-1], B, C, L,
                                     _dtype_code(proj), u.data_ptr(), dc.data_ptr(), _ptr(dc_rev), _stream()),
               "mixer_bwd_prep")
    return (u, dc, dc_rev) if reversed_dc else (u, dc)


def two_stage_taps_grad(dc: torch.Tensor, u: torch.Tensor, lh: int, group_size: int = 1) -> torch.Tensor:
    """dtaps (G, lh) fp32 = sum_{c in g, b, t} dc[t] u[t-j] on tcgen05 (hy_two_stage_taps_grad;
    the two-pass filter gradient of blockconv.py:246-262), bf16 dc / u, lh <= 129."""
    dc3, u3 = _as3(dc), _as3(u)
    _check_device(dc3, u3)
    if dc3.shape != u3.shape or dc3.dtype != torch.bfloat16 or u3.dtype != torch.bfloat16:
        raise ValueError("dc and u must be matching bfloat16 (B, C, L) tensors")
    B, C, L = dc3.shape
    if C % group_size:
        raise ValueError(f"group_size {group_size} does not divide channel count {C}")
    lib = _lib.load()
    out = torch.empty((C // group_size, lh), dtype=torch.float32, device=dc3.device)
    ws = torch.empty(int(lib.hy_two_stage_taps_grad_workspace_size(C, lh)), dtype=torch.uint8, device=dc3.device)
    _lib.check(lib.hy_two_stage_taps_grad(dc3.data_ptr(), u3.data_ptr(), out.data_ptr(), B, C, L, lh, group_size,
                                          _lib.HY_BF16, ws.data_ptr(), ws.numel(), _stream()), "two_stage_taps_grad")
    return out


def featurize(proj: torch.Tensor, feat_taps: torch.Tensor, rhist=None):
    """(u, fq) = ((Fk conv pk) * (Fv conv pv), Fq conv pq) from the (B, 3C, L) projections in
    one stream (hy_featurize_fwd); rhist: optional (B, 3C, 8) raw steps before t = 0."""
    _check_device(proj, rhist)
    B, C3, L = proj.shape
    C = C3 // 3
    if rhist is not None and (tuple(rhist.shape) != (B, C3, 8) or rhist.dtype != proj.dtype):
        raise ValueError(f"rhist must be ({B}, {C3}, 8) {proj.dtype}")
    ft = feat_taps.to(device=proj.device, dtype=torch.float32).contiguous()
    u = torch.empty((B, C, L), dtype=proj.dtype, device=proj.device)
    fq = torch.empty_like(u)
    lib = _lib.load()
    _lib.check(lib.hy_featurize_fwd(proj.data_ptr(), _ptr(rhist), ft.data_ptr(), ft.shape[-1], B, C, L,
                                    _dtype_code(proj), u.data_ptr(), fq.data_ptr(), _stream()), "featurize")
    return u, fq
