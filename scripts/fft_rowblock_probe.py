"""Times the FFT conv (cached filter spectra, hy_fft_conv_spec_fwd) at config C3's size for the
channel block size in HY_FFT_ROW_BLOCK (set by the caller); one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops  # noqa: E402

D, L = int(os.environ.get("FFT_D", 4096)), int(os.environ.get("FFT_L", 131072))
GS = int(os.environ.get("FFT_GS", 1))
g = torch.Generator(device="cuda").manual_seed(0)
v, q, k = (torch.randn((1, D, L), device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
taps = torch.randn((D // GS, L), device="cuda", generator=g) / L ** 0.5
spec = ops.fft_spectrum(taps, L)
f = lambda: ops.long_conv(v, taps, GS, q=q, k=k, spectrum=spec)  # noqa: E731
for _ in range(4):
    f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    y = f()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(json.dumps({"row_block": os.environ.get("HY_FFT_ROW_BLOCK", "256"), "gs": GS, "D": D, "L": L, "ms": ms,
                  "hbm_frac": 4 * 2 * D * L / (ms * 1e-3) / 6542.7e9}))
f2 = lambda: ops.fft_conv(v, taps, GS, q=q, k=k)  # noqa: E731  (filter spectra recomputed per call)
f2()
torch.cuda.synchronize()
s.record()
for _ in range(3):
    f2()
e.record()
torch.cuda.synchronize()
ms2 = s.elapsed_time(e) / 3
print(json.dumps({"row_block": os.environ.get("HY_FFT_ROW_BLOCK", "256"), "gs": GS, "path": "fft_conv (no cached spectra)",
                  "ms": ms2, "hbm_frac": 4 * 2 * D * L / (ms2 * 1e-3) / 6542.7e9}))
