"""Timeline of the implicit (LI) tcgen05 pipeline on CTA 0 (HY_TS_TRACE=1): per-tile events."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["HY_TS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import _lib, ops  # noqa: E402

D, L = 4096, int(os.environ.get("TRACE_L", 131072))
g = torch.Generator(device="cuda").manual_seed(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "conv"
res = torch.randn((D, 8), device="cuda", generator=g) / 8
poles = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
if mode == "conv":
    v = torch.randn((1, D, L), device="cuda", dtype=torch.bfloat16, generator=g)
    run = lambda: ops.li_conv(v, res, poles, 1)
else:
    proj = torch.randn((1, 3 * D, L), device="cuda", dtype=torch.bfloat16, generator=g)
    feat = torch.randn((3, D, 7), device="cuda", generator=g) / 3
    packed = ops.feat_pack(feat)
    run = lambda: ops.li_mixer(proj, feat, res, poles, 1, packed=packed)
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 6144)()
_lib.check(_lib.load().hy_debug_two_stage_trace(buf, 6144), "trace")
tr = np.array(buf, dtype=np.int64).reshape(256, 24).astype(np.float64)
n = 256
tr -= tr[0, 0]
EV = {0: "P_got_empty", 11: "P_issued", 1: "C_ffull", 2: "C_uempty", 3: "C_done", 4: "M_start", 7: "M_E_commit",
      8: "M_tf32", 9: "S_efull", 10: "S_done", 5: "E_tfull", 6: "E_done", 16: "M_ufull", 17: "M_tempty",
      18: "M_eempty", 19: "F_start", 20: "F_sready"}
order = [0, 11, 1, 2, 3, 16, 17, 4, 18, 7, 9, 10, 8, 5, 6]
print("tiles 30..34 and 40..44 (cycles):")
for it in list(range(30, 35)) + list(range(40, 45)):
    print(it, " ".join(f"{EV[e]}={tr[it, e]:8.0f}" for e in order))
big = np.diff(tr[20:n, 6])
print("E_done gaps > 2x median at tiles:", [(i + 21, int(v)) for i, v in enumerate(big) if v > 2 * np.median(big)])
for e in order:
    d = np.diff(tr[20:n, e])
    print(f"period {EV[e]:12s} median {np.median(d):7.0f} mean {d.mean():7.0f}")
def st(a, b):
    d = tr[20:n, b] - tr[20:n, a]
    print(f"{EV[a]:>12s} -> {EV[b]:12s} median {np.median(d):7.0f} p90 {np.percentile(d, 90):7.0f}")
for a, b in [(0, 11), (11, 1), (1, 2), (2, 3), (3, 4), (4, 7), (7, 9), (9, 10), (10, 8), (8, 5), (5, 6),
             (16, 17), (17, 4), (4, 18), (18, 7)]:
    st(a, b)
d = tr[21:n, 16] - tr[20:n - 1, 7]
print(f"{'E_commit(j) -> M_ufull(j+1)':30s} median {np.median(d):7.0f}")
