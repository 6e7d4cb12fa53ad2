"""Probe: is the C2 mixer slower inside the step than standalone because the projection GEMM
leaves dirty lines in L2 that are written back while the mixer streams? Times the mixer right
after the W_qkv GEMM, with and without a read-only 512 MB pass in between (which evicts the
GEMM's dirty lines before the mixer starts), and on a clean L2."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01868_b200 as hy  # noqa: E402

cfg = hy.make_hyena_config("MR", 4096, hy.make_rng(0), inner_len=128, block_size=128)
op = hy.HyenaOperator(cfg, torch.bfloat16)
x = torch.randn((4, 4096, 8192), device="cuda", dtype=torch.bfloat16)
junk = torch.empty(256 * 1024 * 1024, device="cuda", dtype=torch.bfloat16)  # 512 MB
junk.fill_(1.0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def run(mode, reps=20):
    ts = []
    for _ in range(reps):
        proj = op.project(x)
        if mode == "purge":
            junk.sum()
        if mode == "clean":
            torch.cuda.synchronize()
            junk.sum()
            proj = proj.clone()  # the mixer then reads lines written by a plain copy, not the GEMM
            junk.sum()
        ev[0].record()
        op.mixer(proj)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ts.sort()
    return ts[len(ts) // 2]


for mode in ("after_gemm", "purge", "clean", "after_gemm"):
    print(f"{mode:12s} mixer median {run(mode):.4f} ms", flush=True)
