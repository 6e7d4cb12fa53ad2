"""numpy restatement of the reference convhybrid hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates; paths are relative to
/root/reference/pkg/src/convhybrid/. Arithmetic follows the reference exactly:
float64 everywhere, with float32 rounding only at the stage boundaries the
reference rounds at (SeqTensor(..., dtype) constructions). Parameters are plain
numpy arrays / tuples so the oracle does not depend on the product package.

Filter specs (restating core.py:63-137):
    ("explicit", taps)
    ("regularized", taps_hat, decay_rate, base)
    ("implicit", residues, poles, length)
A bank (restating GroupSpec, core.py:161-204) is a dict
    {"channels": d, "group_size": g, "filters": [spec, ...]}.
"""

from __future__ import annotations

import math

import numpy as np

F64 = np.float64
F32 = np.float32

# --------------------------------------------------------------------------
# rng (rand.py:12-15)


def make_rng(seed: int, stream: int = 0) -> np.random.Generator:
    """Philox keyed by seed + stream * golden-ratio constant (rand.py:12-15)."""
    key = (int(seed) + int(stream) * 0x9E3779B97F4A7C15) % (1 << 64)
    return np.random.Generator(np.random.Philox(key=key))


def rel_err(a, b) -> float:
    """||a-b||_inf / max(||b||_inf, 1) (testing.py:57-62)."""
    a = np.asarray(a, dtype=F64)
    b = np.asarray(b, dtype=F64)
    if a.size == 0:
        return 0.0
    denom = max(float(np.max(np.abs(b))), 1.0)
    return float(np.max(np.abs(a - b)) / denom)


# --------------------------------------------------------------------------
# filters (core.py:140-158)


def filter_len(spec) -> int:
    kind = spec[0]
    if kind == "explicit":
        return int(np.asarray(spec[1]).size)
    if kind == "regularized":
        return int(np.asarray(spec[1]).size)
    if kind == "implicit":
        return int(spec[3])
    raise TypeError(f"not a filter spec: {kind!r}")


def materialize(spec) -> np.ndarray:
    """Flat float64 taps (core.py:140-152).

    explicit: copy; regularized: taps_hat * base**(-rate*t) (core.py:145-146);
    implicit: (poles**t) @ residues with 0**0 = 1 (core.py:147-151).
    """
    kind = spec[0]
    if kind == "explicit":
        return np.array(spec[1], dtype=F64)
    if kind == "regularized":
        taps_hat = np.asarray(spec[1], dtype=F64)
        t = np.arange(taps_hat.size, dtype=F64)
        return taps_hat * float(spec[3]) ** (-float(spec[2]) * t)
    if kind == "implicit":
        residues = np.asarray(spec[1], dtype=F64)
        poles = np.asarray(spec[2], dtype=F64)
        t = np.arange(int(spec[3]), dtype=F64)
        powers = poles[None, :] ** t[:, None]
        return powers @ residues
    raise TypeError(f"not a filter spec: {kind!r}")


def bank_taps(bank) -> np.ndarray:
    """(n_groups, lh) tap matrix (GroupSpec.materialized, core.py:198-200)."""
    return np.stack([materialize(f) for f in bank["filters"]])


def bank_taps_per_channel(bank) -> np.ndarray:
    """(channels, lh) (GroupSpec.taps_per_channel, core.py:202-204)."""
    return np.repeat(bank_taps(bank), bank["group_size"], axis=0)


def bank_filter_len(bank) -> int:
    return filter_len(bank["filters"][0])


def explicit_bank(channels: int, group_size: int, taps_list) -> dict:
    return {"channels": channels, "group_size": group_size,
            "filters": [("explicit", np.asarray(t, dtype=F64)) for t in taps_list]}


def uniform_bank(channels: int, taps) -> dict:
    """One shared explicit filter (uniform_groups, core.py:207-209)."""
    return explicit_bank(channels, channels, [taps])


# --------------------------------------------------------------------------
# direct causal conv (core.py:212-226)


def _round(a: np.ndarray, dtype) -> np.ndarray:
    return np.asarray(a, dtype=dtype)


def direct_causal_conv(x: np.ndarray, bank: dict) -> np.ndarray:
    """Per-channel np.convolve(x, h)[:L] in f64, cast to x.dtype (core.py:212-226)."""
    x = np.asarray(x)
    dtype = F32 if x.dtype == F32 else F64
    if x.shape[0] != bank["channels"]:
        raise ValueError(f"input has {x.shape[0]} channels, grouping expects {bank['channels']}")
    taps = bank_taps(bank)
    gs = bank["group_size"]
    out = np.empty(x.shape, dtype=F64)
    for ch in range(x.shape[0]):
        out[ch] = np.convolve(np.asarray(x[ch], dtype=F64), taps[ch // gs])[: x.shape[1]]
    return _round(out, dtype)


def full_toeplitz(h, length: int) -> np.ndarray:
    """T[t,k] = h[t-k] on the band (core.py:229-242)."""
    h = np.asarray(h, dtype=F64)
    idx = np.arange(length)[:, None] - np.arange(length)[None, :]
    mask = (idx >= 0) & (idx < h.size)
    return np.where(mask, h[np.clip(idx, 0, h.size - 1)], 0.0)


# --------------------------------------------------------------------------
# blocked conv (blockconv.py)


def spill_count(lh: int, lb: int) -> int:
    """ceil((lh-1)/lb) (blockconv.py:54-56)."""
    return math.ceil((lh - 1) / lb)


def build_factors(taps, lb: int) -> np.ndarray:
    """(K+1, lb, lb) factors, B_k[i,j] = h[k*lb+i-j] masked to [0, lh) (blockconv.py:59-74)."""
    taps = np.asarray(taps, dtype=F64)
    lh = taps.size
    k_count = spill_count(lh, lb)
    i = np.arange(lb)[:, None]
    j = np.arange(lb)[None, :]
    blocks = np.zeros((k_count + 1, lb, lb))
    for k in range(k_count + 1):
        lag = k * lb + i - j
        valid = (lag >= 0) & (lag < lh)
        blocks[k][valid] = taps[lag[valid]]
    return blocks


def _chunk(arr: np.ndarray, lb: int) -> np.ndarray:
    """(d, l) -> (n, lb, d), zero tail (blockconv.py:89-94)."""
    d, length = arr.shape
    n = math.ceil(length / lb)
    padded = np.zeros((d, n * lb), dtype=arr.dtype)
    padded[:, :length] = arr
    return padded.reshape(d, n, lb).transpose(1, 2, 0)


def _unchunk(chunks: np.ndarray, length: int) -> np.ndarray:
    """(blockconv.py:97-100)."""
    n, lb, d = chunks.shape
    return chunks.transpose(2, 0, 1).reshape(d, n * lb)[:, :length]


def block_conv(x: np.ndarray, bank: dict, lb: int) -> np.ndarray:
    """K-block conv, any lh; output cast to x.dtype (blockconv.py:103-121)."""
    x = np.asarray(x)
    dtype = F32 if x.dtype == F32 else F64
    d, length = x.shape
    gs = bank["group_size"]
    out = np.empty((d, length))
    for g, spec in enumerate(bank["filters"]):
        sl = slice(g * gs, (g + 1) * gs)
        factors = build_factors(materialize(spec), lb)
        chunks = _chunk(np.asarray(x[sl], dtype=F64), lb)
        acc = np.zeros_like(chunks)
        for k in range(min(factors.shape[0] - 1, chunks.shape[0] - 1) + 1):
            if k == 0:
                acc += factors[0] @ chunks
            else:
                acc[k:] += factors[k] @ chunks[:-k]
        out[sl] = _unchunk(acc, length)
    return _round(out, dtype)


class TwoStageIneligibleError(ValueError):
    """K > 1 (blockconv.py:27-28)."""


def _two_factor(taps, lb):
    """(blockconv.py:132-136)."""
    f = build_factors(taps, lb)
    return f[0], (f[1] if f.shape[0] > 1 else np.zeros_like(f[0]))


def two_stage_core(u: np.ndarray, bank: dict, lb: int) -> np.ndarray:
    """Y_n = B0 U_n + B1 U_{n-1}, U_{-1} = 0, per group (blockconv.py:160-179)."""
    d, length = u.shape
    gs = bank["group_size"]
    out = np.empty((d, length))
    for g, spec in enumerate(bank["filters"]):
        sl = slice(g * gs, (g + 1) * gs)
        b0, b1 = _two_factor(materialize(spec), lb)
        chunks = _chunk(u[sl], lb)
        prev = np.concatenate([np.zeros_like(chunks[:1]), chunks[:-1]])
        out[sl] = _unchunk(b0 @ chunks + b1 @ prev, length)
    return out


def two_stage_forward(v: np.ndarray, bank: dict, lb: int, q=None, k=None) -> np.ndarray:
    """y = q * conv(k * v) with optional gates, cast to v.dtype (blockconv.py:182-220)."""
    v = np.asarray(v)
    dtype = F32 if v.dtype == F32 else F64
    if v.shape[0] != bank["channels"]:
        raise ValueError(f"input has {v.shape[0]} channels, grouping expects {bank['channels']}")
    for name, gate in (("q", q), ("k", k)):
        if gate is not None and np.shape(gate) != v.shape:
            raise ValueError(f"gate {name} shape {np.shape(gate)} does not match input {v.shape}")
    if spill_count(bank_filter_len(bank), lb) > 1:
        raise TwoStageIneligibleError("filter needs more than one spill factor")
    u = np.asarray(v, dtype=F64)
    if k is not None:
        u = u * np.asarray(k, dtype=F64)
    c = two_stage_core(u, bank, lb)
    y = c * np.asarray(q, dtype=F64) if q is not None else c
    return _round(y, dtype)


def chunk_parallel_forward(v: np.ndarray, taps, lb: int) -> np.ndarray:
    """All chunks as GEMM columns, one shared filter (blockconv.py:267-293)."""
    v = np.asarray(v)
    dtype = F32 if v.dtype == F32 else F64
    taps = np.asarray(taps, dtype=F64)
    if spill_count(taps.size, lb) > 1:
        raise TwoStageIneligibleError("filter needs more than one spill factor")
    b0, b1 = _two_factor(taps, lb)
    chunks = _chunk(np.asarray(v, dtype=F64), lb)
    n, _, d = chunks.shape
    cols = chunks.transpose(1, 0, 2).reshape(lb, n * d)
    prev = np.concatenate([np.zeros_like(chunks[:1]), chunks[:-1]])
    prev_cols = prev.transpose(1, 0, 2).reshape(lb, n * d)
    out_cols = b0 @ cols + b1 @ prev_cols
    out = _unchunk(out_cols.reshape(lb, n, d).transpose(1, 0, 2), v.shape[1])
    return _round(out, dtype)


def two_stage_flops(length: int, lb: int, channels: int) -> int:
    """2 * lb^2 * d * ceil(l/lb) (blockconv.py:296-300)."""
    return 2 * lb * lb * channels * math.ceil(length / lb)


# --------------------------------------------------------------------------
# radix-2 FFT (fft.py)


def next_pow2(n: int) -> int:
    """(fft.py:30-34)."""
    if n < 1:
        raise ValueError(f"need n >= 1, got {n}")
    return 1 << (n - 1).bit_length()


def bit_reversal_indices(l: int) -> np.ndarray:
    """(fft.py:55-63)."""
    bits = l.bit_length() - 1
    idx = np.arange(l)
    rev = np.zeros(l, dtype=np.int64)
    for _ in range(bits):
        rev = (rev << 1) | (idx & 1)
        idx >>= 1
    return rev


def _dif_passes(x: np.ndarray) -> np.ndarray:
    """All DiF butterflies, natural in -> bit-reversed out (fft.py:100-113)."""
    z = np.array(x, dtype=np.complex128, copy=True)
    l = z.shape[-1]
    span = l // 2
    while span >= 1:
        blocks = z.reshape(z.shape[:-1] + (-1, 2, span))
        lo = blocks[..., 0, :].copy()
        hi = blocks[..., 1, :]
        w = np.exp(-2j * np.pi * np.arange(span) / (2 * span))
        blocks[..., 0, :] = lo + hi
        blocks[..., 1, :] = (lo - hi) * w
        span //= 2
    return z


def fft(x) -> np.ndarray:
    """(fft.py:116-118)."""
    z = _dif_passes(x)
    return z[..., bit_reversal_indices(z.shape[-1])]


def ifft(y) -> np.ndarray:
    """conj(fft(conj(y))) / l (fft.py:121-125)."""
    y = np.asarray(y, dtype=np.complex128)
    return np.conj(fft(np.conj(y))) / y.shape[-1]


def dft_oracle(x) -> np.ndarray:
    """O(l^2) DFT (fft.py:37-43)."""
    x = np.asarray(x, dtype=np.complex128)
    l = x.shape[-1]
    jk = np.arange(l)[:, None] * np.arange(l)[None, :]
    return x @ np.exp(-2j * np.pi * jk / l)


def fft_conv(x, taps) -> np.ndarray:
    """Zero-padded causal conv via radix-2 FFT, f64 result (fft.py:128-145)."""
    x = np.asarray(x, dtype=F64)
    taps = np.asarray(taps, dtype=F64)
    l = x.shape[-1]
    lh = taps.shape[-1]
    size = next_pow2(max(l + lh - 1, 1))
    xp = np.zeros(x.shape[:-1] + (size,))
    xp[..., :l] = x
    hp = np.zeros(taps.shape[:-1] + (size,))
    hp[..., :lh] = taps
    spec = fft(xp) * fft(hp)
    return ifft(spec).real[..., :l]


# --------------------------------------------------------------------------
# Hyena operator (hyena.py)

VARIANTS = ("SE", "MR", "LI")
MAX_SHORT_FILTER = 14


def projection_dense(p) -> np.ndarray:
    """(hyena.py:64-65)."""
    return p[0] @ p[1] if isinstance(p, tuple) else np.asarray(p, dtype=F64)


def _featurize(xd: np.ndarray, proj, bank: dict, dtype):
    """a = W^T x (f64), conv on a rounded to dtype, featurized back to f64 (hyena.py:122-126)."""
    a = projection_dense(proj).T @ xd
    b = direct_causal_conv(_round(a, dtype), bank)
    return np.asarray(b, dtype=F64)


def _inner_conv(u: np.ndarray, cfg: dict, dtype) -> np.ndarray:
    """Backend dispatch (hyena.py:129-135): direct/blocked round u to dtype; fft does not."""
    if cfg["backend"] == "direct":
        return np.asarray(direct_causal_conv(_round(u, dtype), cfg["inner"]), dtype=F64)
    if cfg["backend"] == "blocked":
        return np.asarray(block_conv(_round(u, dtype), cfg["inner"], cfg["block_size"]), dtype=F64)
    return fft_conv(u, bank_taps_per_channel(cfg["inner"]))


def hyena_forward(x: np.ndarray, cfg: dict) -> np.ndarray:
    """Eq. 1: y = W_out^T (q * conv_inner(k * v)) (hyena.py:157-190)."""
    x = np.asarray(x)
    dtype = F32 if x.dtype == F32 else F64
    if x.shape[0] != cfg["width"]:
        raise ValueError(f"input has {x.shape[0]} channels, operator width is {cfg['width']}")
    lh = bank_filter_len(cfg["inner"])
    if cfg["variant"] == "LI" and lh != x.shape[1]:
        raise ValueError(f"LI inner filter length {lh} must equal the sequence length {x.shape[1]}")
    xd = np.asarray(x, dtype=F64)
    q = _featurize(xd, cfg["w_q"], cfg["q_feat"], dtype)
    k = _featurize(xd, cfg["w_k"], cfg["k_feat"], dtype)
    v = _featurize(xd, cfg["w_v"], cfg["v_feat"], dtype)
    if cfg["backend"] == "blocked" and spill_count(lh, cfg["block_size"]) <= 1:
        # two_stage_forward_saved(SeqTensor(v, dtype), ..., q=..., k=...) (hyena.py:175-182)
        u = v * k
        c = two_stage_core(u, cfg["inner"], cfg["block_size"])
        mixed = np.asarray(_round(c * q, dtype), dtype=F64)
    else:
        gated = k * v  # (hyena.py:184-186)
        conv_out = _inner_conv(gated, cfg, dtype)
        mixed = q * conv_out
    y = projection_dense(cfg["w_out"]).T @ mixed
    return _round(y, dtype)


def layout_forward(x: np.ndarray, layers, residual: bool = False) -> np.ndarray:
    """Sequential stack with optional residual (hyena.py:394-406)."""
    x = np.asarray(x)
    dtype = F32 if x.dtype == F32 else F64
    cur = x
    for cfg in layers:
        out = hyena_forward(cur, cfg)
        cur = _round(np.asarray(cur, dtype=F64) + np.asarray(out, dtype=F64), dtype) if residual else out
    return cur


# --------------------------------------------------------------------------
# seeded builders (hyena.py:423-533) — identical draw order to the reference

DEFAULT_FEATURIZER_LEN = 7
DEFAULT_SE_LEN = 7
DEFAULT_MR_LEN = 128
DEFAULT_LI_POLES = 8
DECAY_SWEEP = (0.01, 2.0)


def _rand_taps(rng, lh):
    """N(0, 1/lh) taps (hyena.py:430-431)."""
    return rng.standard_normal(lh) / np.sqrt(lh)


def _explicit_bank(rng, width, group_size, lh):
    """(hyena.py:434-436)."""
    n = width // group_size
    return {"channels": width, "group_size": group_size,
            "filters": [("explicit", _rand_taps(rng, lh)) for _ in range(n)]}


def make_inner_bank(variant, width, group_size, rng, filter_len=None, seq_len=None,
                    n_poles=DEFAULT_LI_POLES, decay_base=2.0):
    """(hyena.py:439-469)."""
    n = width // group_size
    if variant == "SE":
        return _explicit_bank(rng, width, group_size, DEFAULT_SE_LEN if filter_len is None else filter_len)
    if variant == "MR":
        lh = DEFAULT_MR_LEN if filter_len is None else filter_len
        rates = np.linspace(DECAY_SWEEP[0], DECAY_SWEEP[1], n)
        return {"channels": width, "group_size": group_size,
                "filters": [("regularized", _rand_taps(rng, lh), float(rates[g]), decay_base)
                            for g in range(n)]}
    if variant == "LI":
        if seq_len is None:
            raise ValueError("LI inner filters need the sequence length")
        filters = []
        for _ in range(n):
            poles = rng.uniform(-0.95, 0.95, size=n_poles)
            residues = rng.standard_normal(n_poles) / n_poles
            filters.append(("implicit", residues, poles, seq_len))
        return {"channels": width, "group_size": group_size, "filters": filters}
    raise ValueError(f"variant must be one of {VARIANTS}, got {variant!r}")


def make_hyena_config(variant, width, rng, seq_len=None, group_size=1,
                      featurizer_len=DEFAULT_FEATURIZER_LEN, inner_len=None, block_size=16,
                      backend="blocked", n_poles=DEFAULT_LI_POLES) -> dict:
    """(hyena.py:472-497); returns the oracle's dict form of HyenaConfig."""
    scale = 1.0 / np.sqrt(width)
    projs = [rng.standard_normal((width, width)) * scale for _ in range(4)]
    return {
        "variant": variant, "width": width,
        "w_q": projs[0], "w_k": projs[1], "w_v": projs[2], "w_out": projs[3],
        "q_feat": _explicit_bank(rng, width, group_size, featurizer_len),
        "k_feat": _explicit_bank(rng, width, group_size, featurizer_len),
        "v_feat": _explicit_bank(rng, width, group_size, featurizer_len),
        "inner": make_inner_bank(variant, width, group_size, rng, filter_len=inner_len,
                                 seq_len=seq_len, n_poles=n_poles),
        "block_size": block_size, "backend": backend,
    }


def identity_config(variant="SE", width=1, inner=None, backend="direct", block_size=16) -> dict:
    """(hyena.py:516-533)."""
    eye = np.eye(width)
    unit = uniform_bank(width, [1.0])
    return {"variant": variant, "width": width, "w_q": eye, "w_k": eye.copy(), "w_v": eye.copy(),
            "w_out": eye.copy(), "q_feat": unit, "k_feat": unit, "v_feat": unit,
            "inner": unit if inner is None else inner, "block_size": block_size, "backend": backend}
