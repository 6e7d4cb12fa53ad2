"""The reference's fft module API on the device (fft.py:24-157), mirroring the reference's
own test_fft.py cases: DFT oracles, bit reversal, DiF split / DiT merge, FFT vs the O(l^2)
oracle, linearity, round trip, Parseval, circular-conv oracle, fft_conv."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2503_01868_b200 import fft

pytestmark = pytest.mark.gpu


def test_dft_oracles_known_answers():
    l = 8
    delta = np.zeros(l)
    delta[0] = 1.0
    assert np.allclose(fft.dft_oracle(delta), np.ones(l), atol=1e-14)
    assert np.allclose(fft.dft_oracle(np.ones(l)), l * delta, atol=1e-12)
    tone = np.exp(2j * np.pi * 3 * np.arange(l) / l)
    want = np.zeros(l, dtype=complex)
    want[3] = l
    assert np.allclose(fft.dft_oracle(tone), want, atol=1e-12)
    x = np.random.default_rng(1).standard_normal((3, 16))
    assert np.allclose(fft.idft_oracle(fft.dft_oracle(x)), x, atol=1e-12)


def test_bit_reversal():
    assert list(fft.bit_reversal_indices(8)) == [0, 4, 2, 6, 1, 5, 3, 7]
    x = np.random.default_rng(2).standard_normal((2, 3, 32))
    assert np.array_equal(fft.bit_reversal(fft.bit_reversal(x)), x)
    assert np.array_equal(fft.bit_reversal(x)[1, 2], x[1, 2][fft.bit_reversal_indices(32)])
    with pytest.raises(ValueError):
        fft.bit_reversal_indices(12)


def test_dif_split_and_dit_merge():
    x = np.random.default_rng(3).standard_normal((2, 16)) + 1j * np.random.default_rng(4).standard_normal((2, 16))
    a, b = fft.dif_split(x)
    full = fft.dft_oracle(x)
    assert np.allclose(fft.dft_oracle(a), full[..., 0::2], atol=1e-12)
    assert np.allclose(fft.dft_oracle(b), full[..., 1::2], atol=1e-12)
    assert np.allclose(fft.dit_merge(a, b), x, atol=1e-14)
    with pytest.raises(ValueError):
        fft.dit_merge(a, b[..., :4])
    with pytest.raises(ValueError):
        fft.dif_split(np.ones(1))


@pytest.mark.parametrize("l", [1, 2, 8, 64, 1024])
def test_fft_matches_oracle_and_roundtrips(l):
    rng = np.random.default_rng(l)
    x = rng.standard_normal((3, l)) + 1j * rng.standard_normal((3, l))
    y = fft.fft(x)
    assert np.allclose(y, fft.dft_oracle(x), atol=1e-9 * max(1, l))
    assert np.allclose(fft.bit_reversal(fft._dif_passes(x)), y, atol=1e-9 * max(1, l))
    assert np.allclose(fft.ifft(y), x, atol=1e-12)
    # linearity, Parseval, normalisation on the inverse side
    z = rng.standard_normal((3, l))
    assert np.allclose(fft.fft(2 * x + z), 2 * y + fft.fft(z), atol=1e-9 * max(1, l))
    assert np.allclose((np.abs(y) ** 2).sum(-1) / l, (np.abs(x) ** 2).sum(-1))
    assert np.allclose(fft.fft(np.ones(l)).real[0], l)


def test_fft_rejects_non_pow2():
    with pytest.raises(ValueError):
        fft.fft(np.ones(12))
    with pytest.raises(ValueError):
        fft.ifft(np.ones(6))


def test_circular_conv_oracle():
    rng = np.random.default_rng(5)
    x = rng.standard_normal(8)
    delta = np.zeros(8)
    delta[0] = 1.0
    assert np.allclose(fft.circular_conv_oracle(x, delta), x)
    shift = np.zeros(8)
    shift[1] = 1.0
    assert np.allclose(fft.circular_conv_oracle(x, shift), np.roll(x, 1))  # wraps
    h = rng.standard_normal(8)
    assert np.allclose(fft.circular_conv_oracle(x, h), fft.ifft(fft.fft(x) * fft.fft(h)).real, atol=1e-12)
    with pytest.raises(ValueError):
        fft.circular_conv_oracle(x, h[:4])


def test_fft_conv_matches_direct():
    rng = np.random.default_rng(6)
    x = rng.standard_normal((3, 100))
    taps = rng.standard_normal(17)
    y = fft.fft_conv(x, taps)
    want = oracle.direct_causal_conv(x, {"channels": 3, "group_size": 3, "filters": [("explicit", taps)]})
    assert y.shape == x.shape and y.dtype == np.float64
    assert np.max(np.abs(y - want)) < 1e-10
    per = rng.standard_normal((3, 9))
    y = fft.fft_conv(x, per)
    want = oracle.direct_causal_conv(x, {"channels": 3, "group_size": 1, "filters": [("explicit", t) for t in per]})
    assert np.max(np.abs(y - want)) < 1e-10
    long = rng.standard_normal(150)  # filter longer than the sequence
    want = oracle.direct_causal_conv(x, {"channels": 3, "group_size": 3, "filters": [("explicit", long)]})
    assert np.max(np.abs(fft.fft_conv(x, long) - want)) < 1e-10


@pytest.mark.parametrize("dtype", [torch.complex128, torch.complex64])
@pytest.mark.parametrize("n,batch", [(1, 3), (2, 5), (1024, 7), (8192, 2), (16384, 2), (1 << 18, 2)])
def test_fft_c2c_kernel_vs_dft(dtype, n, batch):
    """hy_fft_c2c (radix-2 Stockham; shared-memory rows and the multi-pass global path) against
    the oracle's radix-2 DiF transform in float64 (fft.py:100-125): forward unnormalised,
    inverse with 1/n; complex64 within fp32 rounding, complex128 within 1e-12."""
    from paper_2503_01868_b200 import ops
    rng = np.random.default_rng(n + batch)
    x = rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))
    xd = torch.from_numpy(x).to("cuda", dtype)
    y = ops.fft_c2c(xd).cpu().numpy()
    want = oracle.fft(x.astype(np.complex64 if dtype == torch.complex64 else np.complex128))
    tol = 1e-12 if dtype == torch.complex128 else 1e-5

    def cerr(a, b):  # rel_err (testing.py:57-62) on complex values: inf-norm of the difference
        return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1.0))
    assert cerr(y, want) < tol
    back = ops.fft_c2c(torch.from_numpy(y).to("cuda", dtype), inverse=True).cpu().numpy()
    assert cerr(back, x) < tol
