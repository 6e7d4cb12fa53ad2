"""LI mixer timeline inside the operator step (projection GEMM right before it) vs standalone."""
import ctypes, os, sys
import numpy as np
import torch
os.environ["HY_TS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import _lib, ops

D, L = 4096, 131072
cfg = hy.make_hyena_config("LI", D, hy.make_rng(0), seq_len=L)
op = hy.HyenaOperator(cfg, torch.bfloat16)
x = torch.randn((1, D, L), device="cuda").to(torch.bfloat16)

def trace():
    buf = (ctypes.c_ulonglong * 6144)()
    _lib.check(_lib.load().hy_debug_two_stage_trace(buf, 6144), "trace")
    tr = np.array(buf, dtype=np.int64).reshape(256, 24).astype(np.float64)
    d = np.diff(tr[20:256, 6])
    return np.median(d), d.mean(), (tr[255, 6] - tr[20, 6])

for mode in ("standalone", "in-step", "standalone", "in-step"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    proj = op.project(x)
    torch.cuda.synchronize()
    if mode == "in-step":
        for _ in range(3):
            op.forward(x)
        proj = op.project(x)  # GEMM immediately before the mixer
        ev[0].record()
        m = op.mixer(proj)
        ev[1].record()
    else:
        torch.cuda.synchronize()
        ev[0].record()
        m = op.mixer(proj)
        ev[1].record()
    torch.cuda.synchronize()
    med, mean, span = trace()
    print(f"{mode:10s} mixer {ev[0].elapsed_time(ev[1]):.3f} ms  tile period median {med:.0f} mean {mean:.0f} cycles, span {span:.0f}")
