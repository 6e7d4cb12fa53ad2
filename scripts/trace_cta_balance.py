"""Per-CTA start / end times (globaltimer) of one traced two_stage_kernel launch (the fused LI or
MR mixer, HY_TS_TRACE=1): how evenly the persistent CTAs finish.
Usage: TRACE_L=16384 python scripts/trace_cta_balance.py mixer|mr"""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["HY_TS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import _lib, ops  # noqa: E402

D, L = 4096, int(os.environ.get("TRACE_L", 16384))
g = torch.Generator(device="cuda").manual_seed(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "mixer"
res = torch.randn((D, 8), device="cuda", generator=g) / 8
poles = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
proj = torch.randn((1, 3 * D, L), device="cuda", dtype=torch.bfloat16, generator=g)
feat = torch.randn((3, D, 7), device="cuda", generator=g) / 3
packed = ops.feat_pack(feat)
taps = torch.randn((D, 128), device="cuda", generator=g) / 11
if mode == "mixer":
    run = lambda: ops.li_mixer(proj, feat, res, poles, 1, packed=packed)  # noqa: E731
else:
    run = lambda: ops.hyena_mixer(proj, feat, taps, 1, packed=packed)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
nt = 256 * 24
buf = (ctypes.c_ulonglong * (nt + 512))()
_lib.check(_lib.load().hy_debug_two_stage_trace(buf, nt + 512), "trace")
ct = np.array(buf[nt:], dtype=np.int64).reshape(256, 2)[:148].astype(np.float64)
t0 = ct[:, 0].min()
st, en = (ct[:, 0] - t0) / 1e3, (ct[:, 1] - t0) / 1e3
print(f"{mode} L={L}: start spread {st.max():.1f} us; end min {en.min():.1f} median {np.median(en):.1f} "
      f"max {en.max():.1f} us; slowest CTAs {np.argsort(en)[-8:].tolist()}; fastest {np.argsort(en)[:8].tolist()}")
print("end times (us), CTA order:", " ".join(f"{v:.0f}" for v in en))
