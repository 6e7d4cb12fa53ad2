"""Backward-pass timing at the BASELINE configs (device-resident, CUDA events, after warm-up):
the whole operator_backward step and its conv kernels alone. Tuning aid; bench.py
--workload mr_train is the contract line."""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_01868_b200 as hy  # noqa: E402
from paper_2503_01868_b200 import ops  # noqa: E402


def timeit(fn, iters=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def cfg_for(variant, D, L):
    kw = {"seq_len": L} if variant == "LI" else {"inner_len": 128 if variant == "MR" else 7}
    return hy.make_hyena_config(variant, D, hy.make_rng(0), block_size=128 if variant == "MR" else 16, **kw)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="mr,se,li")
    ap.add_argument("--profile", action="store_true")
    args = ap.parse_args()
    hy.hyena._fp32_exact()
    confs = {"mr": ("MR", 4, 8192, torch.bfloat16), "se": ("SE", 1, 4096, torch.float32),
             "li": ("LI", 1, 131072, torch.bfloat16)}
    for key in args.which.split(","):
        variant, B, L, dt = confs[key]
        D = 4096
        op = hy.HyenaOperator(cfg_for(variant, D, L), dt)
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.randn((B, D, L), device="cuda", dtype=dt, generator=g)
        dy = torch.randn((B, D, L), device="cuda", dtype=dt, generator=g)
        fwd = timeit(lambda: op.forward(x))
        bwd = timeit(lambda: hy.operator_backward(op, x, dy))
        esz = x.element_size()
        out = {"workload": key, "B": B, "L": L, "dtype": str(dt), "fwd_ms": round(fwd, 3), "bwd_ms": round(bwd, 3)}
        u = torch.randn((B, D, L), device="cuda", dtype=dt, generator=g)
        if variant == "MR" and dt == torch.bfloat16:
            ms = timeit(lambda: ops.two_stage_taps_grad(dy, u, 128, 1))
            out["taps_grad_tcgen05_ms"] = round(ms, 3)
            out["taps_grad_tcgen05_GBps"] = round(2 * B * D * L * esz / ms / 1e6, 1)
        if variant != "LI":
            taps = op.materialized_inner
            ms = timeit(lambda: ops.causal_conv_bwd(dy, u, taps, 1))
            out["inner_conv_bwd_ms"] = round(ms, 3)
            out["inner_conv_bwd_GBps"] = round(3 * B * D * L * esz / ms / 1e6, 1)
            out["inner_conv_bwd_TFLOPs"] = round(4 * taps.shape[-1] * B * D * L / ms / 1e9, 2)
        else:
            r = torch.randn((D, 8), device="cuda", generator=g) / 8
            p = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
            ms = timeit(lambda: ops.li_param_grad(dy, u, r, p, 1))
            out["li_param_grad_ms"] = round(ms, 3)
            out["li_param_grad_GBps"] = round(2 * B * D * L * esz / ms / 1e6, 1)
        proj = torch.randn((B, 3 * D, L), device="cuda", dtype=dt, generator=g)
        ms = timeit(lambda: ops.featurizer_bwd(proj, dy, u, x, op.feat_taps))
        out["featurizer_bwd_ms"] = round(ms, 3)
        out["featurizer_bwd_GBps"] = round(9 * B * D * L * esz / ms / 1e6, 1)  # 6 rows in, 3 out
        print(json.dumps(out), flush=True)
        if args.profile:
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                hy.operator_backward(op, x, dy)
                torch.cuda.synchronize()
            print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25), flush=True)
        del op, x, dy, u, proj
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
