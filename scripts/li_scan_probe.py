"""Times the modal-scan LI mixer (hy_li_scan_mixer_fwd) and gated conv (hy_li_scan_fwd) at config
C3's size in fp32 (the reference's precision); one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops  # noqa: E402

D, L = 4096, int(os.environ.get("LIS_L", 131072))
g = torch.Generator(device="cuda").manual_seed(0)
proj = torch.randn((1, 3 * D, L), device="cuda", generator=g)
feat = torch.randn((3, D, 7), device="cuda", generator=g) / 2.65
res = (torch.randn((D, 8), device="cuda", generator=g) / 8).double()
poles = (torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95).double()


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


ms_mix = timed(lambda: ops.li_scan_mixer(proj, feat, res, poles, 1))
v, q, k = proj[:, 2 * D:].contiguous(), proj[:, :D].contiguous(), proj[:, D:2 * D].contiguous()
ms_conv = timed(lambda: ops.li_scan(v, res, poles, 1, q=q, k=k))
nb = 4 * 4 * D * L
print(json.dumps({"L": L, "mixer_ms": ms_mix, "mixer_hbm_frac": nb / (ms_mix * 1e-3) / 6542.7e9,
                  "gated_conv_ms": ms_conv, "gated_conv_hbm_frac": nb / (ms_conv * 1e-3) / 6542.7e9}))
