"""MR mixer timeline (CTA 0 cycles) and wall time inside the operator step vs standalone."""
import ctypes, os, sys
import numpy as np
import torch
os.environ["HY_TS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01868_b200 as hy
from paper_2503_01868_b200 import _lib

B, D, L = 4, 4096, 8192
cfg = hy.make_hyena_config("MR", D, hy.make_rng(0), inner_len=128, block_size=128)
op = hy.HyenaOperator(cfg, torch.bfloat16)
x = torch.randn((B, D, L), device="cuda").to(torch.bfloat16)

def trace():
    buf = (ctypes.c_ulonglong * 6144)()
    _lib.check(_lib.load().hy_debug_two_stage_trace(buf, 6144), "trace")
    tr = np.array(buf, dtype=np.int64).reshape(256, 24).astype(np.float64)
    d = np.diff(tr[5:221, 6])
    return np.median(d), d.mean(), tr[220, 6] - tr[5, 6]

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for mode in ("standalone", "in-step", "after-flush", "standalone", "in-step", "after-flush"):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    proj = op.project(x)
    torch.cuda.synchronize()
    if mode == "in-step":
        for _ in range(3):
            op.forward(x)
        proj = op.project(x)
    elif mode == "after-flush":
        proj = op.project(x)
        flush.zero_()  # L2 holds clean flush lines instead of the GEMM's dirty output
    else:
        torch.cuda.synchronize()
    ev[0].record()
    m = op.mixer(proj)
    ev[1].record()
    torch.cuda.synchronize()
    med, mean, span = trace()
    print(f"{mode:11s} mixer {ev[0].elapsed_time(ev[1]):.3f} ms  tile period median {med:.0f} mean {mean:.0f} cycles, span {span:.0f}")
