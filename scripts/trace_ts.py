"""Timeline of the tcgen05 mixer pipeline on CTA 0 (HY_TS_TRACE=1): per-tile event deltas."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["HY_TS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import _lib, ops  # noqa: E402

B, D, L = 4, 4096, 8192
g = torch.Generator(device="cuda").manual_seed(0)
proj = torch.randn((B, 3 * D, L), device="cuda", dtype=torch.bfloat16, generator=g)
feat = torch.randn((3, D, 7), device="cuda", generator=g) / 3
taps = torch.randn((D, 128), device="cuda", generator=g) / 11
mode = sys.argv[1] if len(sys.argv) > 1 else "mixer"
for _ in range(3):
    if mode == "mixer":
        ops.hyena_mixer(proj, feat, taps, 1)
    else:
        v, k, q = (proj[:, i * D:(i + 1) * D].contiguous() for i in range(3))
        ops.two_stage(v, taps, 1, q=q, k=k)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 6144)()
_lib.check(_lib.load().hy_debug_two_stage_trace(buf, 6144), "trace")
tr = np.array(buf, dtype=np.int64).reshape(256, 24)
n = 221
tr = tr[:n].astype(np.float64)
tr -= tr[0, 0]
names = ["P_issue", "C_full", "C_start", "C_done", "M_issue", "E_start", "E_store"]
print("first tiles (cycles since first issue):")
for it in range(8):
    print(it, " ".join(f"{names[e]}={tr[it, e]:9.0f}" for e in range(7)))
per = np.diff(tr[:, 6])
print(f"tiles {n}, total {tr[n-1,6]:.0f} cyc, period(E_store) mean {per[5:].mean():.0f} median {np.median(per[5:]):.0f}")
def st(a, b, lab):
    d = tr[5:, b] - tr[5:, a]
    print(f"{lab:28s} mean {d.mean():8.0f} median {np.median(d):8.0f} p90 {np.percentile(d, 90):8.0f}")
st(0, 1, "load latency (issue->full)")
st(1, 2, "C wait uempty")
st(2, 3, "convert")
st(3, 4, "C_done -> M_issue")
st(4, 5, "MMA issue -> E_start")
st(5, 6, "epilogue")
d = tr[6:, 0] - tr[5:-1, 3]
print(f"{'P_issue(it+1)-C_done(it)':28s} mean {d.mean():8.0f}")

st(0, 7, "P decode")
st(7, 8, "P zero fill")
st(8, 9, "P F build")
st(9, 10, "P fence+syncwarp")
st(10, 11, "P expect+copies")
gc = []
if gc:
    d = np.array([[tr[it, 7] - tr[it, 2], tr[it, 8] - tr[it, 7], tr[it, 9] - tr[it, 8], tr[it, 10] - tr[it, 9],
                   tr[it, 3] - tr[it, 10]] for it in gc])
    print("group-change tiles:", len(gc), "U-build / wait prevMMA / hpad+bar / T build / tail (median):",
          np.median(d, axis=0))

st(12, 0, "P wait empty")
st(0, 11, "P issue (zero/F/copies)")
st(11, 14, "copies land (full)")
st(14, 15, "FMMA wait fempty")
st(15, 13, "FMMA issue")
st(13, 1, "feat MMA -> C sees ffull")
