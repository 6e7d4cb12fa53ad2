"""Kernel micro-benchmarks (device-resident inputs, CUDA events, after warm-up).

Prints one JSON line per kernel: duration, algorithmic bytes, achieved GB/s and
fraction of the measured HBM peak. Used for tuning; bench.py is the contract.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_01868_b200 import ops  # noqa: E402


def peak_hbm():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except OSError:
        return 6650.0


def timeit(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # hold the stream ~10 ms so the host enqueues every iteration before the first one starts:
    # the events then bracket device time, not the per-call host overhead (~tens of us)
    torch.cuda._sleep(20_000_000)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def report(name, ms, nbytes, **extra):
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "bytes": nbytes, "GB/s": round(gbs, 1),
                      "frac_hbm": round(gbs / peak_hbm(), 3), **extra}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="all")
    args = ap.parse_args()
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    # MR mixer at C2: proj (4, 3*4096, 8192) bf16 -> y (4, 4096, 8192)
    if args.which in ("all", "mr"):
        B, D, L = 4, 4096, 8192
        proj = torch.randn((B, 3 * D, L), device=dev, dtype=torch.bfloat16, generator=g)
        feat = torch.randn((3, D, 7), device=dev, generator=g) / 3
        taps = torch.randn((D, 128), device=dev, generator=g) / 11
        decay = torch.linspace(0.01, 2.0, D, device=dev)
        packed = ops.feat_pack(feat)
        ms = timeit(lambda: ops.hyena_mixer(proj, feat, taps, 1, decay=decay, packed=packed))
        report("mr_mixer_tcgen05", ms, 8 * D * B * L, B=B, D=D, L=L)
        v = proj[:, :D].contiguous()
        k = proj[:, D:2 * D].contiguous()
        q = proj[:, 2 * D:].contiguous()
        ms = timeit(lambda: ops.two_stage(v, taps, 1, q=q, k=k, decay=decay))
        report("two_stage_tcgen05_gated", ms, 8 * D * B * L, B=B, D=D, L=L)
        del proj, v, k, q
    if args.which in ("all", "se", "copy"):
        for mb in (134, 537, 2147):  # torch copy with the same total traffic as SE/LI kernels
            n = mb * 1000 * 1000 // 4
            a = torch.empty(n, device=dev, dtype=torch.float32)
            b = torch.empty_like(a)
            ms = timeit(lambda: b.copy_(a))
            report(f"torch_copy_{2 * mb}MB", ms, 2 * n * 4)
            del a, b
    if args.which in ("all", "se"):
        B, D, L = 1, 4096, 4096
        for dt, name in ((torch.float32, "se_mixer_f32"), (torch.bfloat16, "se_mixer_bf16")):
            proj = torch.randn((B, 3 * D, L), device=dev, dtype=dt, generator=g)
            feat = torch.randn((3, D, 7), device=dev, generator=g) / 3
            taps = torch.randn((D, 7), device=dev, generator=g) / 3
            ms = timeit(lambda: ops.hyena_mixer(proj, feat, taps, 1, se_only=True))
            report(name, ms, 4 * D * B * L * proj.element_size(), B=B, D=D, L=L)
            if dt == torch.bfloat16:  # the path the operator takes for bf16 SE: the tcgen05 mixer
                pk = ops.feat_pack(feat)  # packed featurizer factors, built once per weight set
                ms = timeit(lambda: ops.hyena_mixer(proj, feat, taps, 1, packed=pk))
                report("se_mixer_bf16_tcgen05", ms, 4 * D * B * L * proj.element_size(), B=B, D=D, L=L)
            x = proj.reshape(B * 3, D, L)
            ms = timeit(lambda: ops.causal_conv(x, feat.reshape(3 * D, 7), 1))
            report(name.replace("se_mixer", "featurizer"), ms, 2 * x.numel() * x.element_size(), rows=3 * D, L=L)
        for dt, name in ((torch.float32, "se_mixer_f32_B4"),):
            proj = torch.randn((4, 3 * D, L), device=dev, dtype=dt, generator=g)
            ms = timeit(lambda: ops.hyena_mixer(proj, feat, taps, 1, se_only=True))
            report(name, ms, 4 * D * 4 * L * proj.element_size(), B=4, D=D, L=L)
            del proj
    if args.which in ("all", "li"):
        D = 4096
        for L in (131072, 16384):
            proj = torch.randn((1, 3 * D, L), device=dev, dtype=torch.bfloat16, generator=g)
            feat = torch.randn((3, D, 7), device=dev, generator=g) / 3
            packed = ops.feat_pack(feat)
            res = torch.randn((D, 8), device=dev, generator=g) / 8
            poles = torch.rand((D, 8), device=dev, generator=g) * 1.9 - 0.95
            ms = timeit(lambda: ops.li_mixer(proj, feat, res, poles, 1, packed=packed))
            report("li_mixer_tcgen05", ms, 8 * D * L, D=D, L=L)
            v = proj[:, :D]
            ms = timeit(lambda: ops.li_conv(v, res, poles, 1))
            report("li_conv_ungated", ms, 4 * D * L, D=D, L=L)
            del proj, v
        # the CP layer's per-segment slab conv at L = 1M (the all-to-all's rank-major layout):
        # N = 2 / 4 ranks, n_pipe = 4 segments -> 512 / 256 channels of the full sequence
        for n in (2, 4):
            C, m = D // (4 * n), (1 << 20) // n
            buf = torch.randn((n, C, m), device=dev, dtype=torch.bfloat16, generator=g)
            res = torch.randn((C, 8), device=dev, generator=g) / 8
            poles = torch.rand((C, 8), device=dev, generator=g) * 1.9 - 0.95
            ms = timeit(lambda: ops.li_conv_segmented(buf, res, poles, 1))
            report(f"li_conv_segmented_cp{n}", ms, 4 * C * (1 << 20), C=C, L=1 << 20, n_seg=n)
            del buf
    if args.which in ("all", "scan"):
        # modal-scan LI kernels (CUDA cores) at C3: fp32 mixer (the reference precision), bf16
        # ungated conv (vs li_conv_ungated above) and the bf16 mixer
        D, L = 4096, 131072
        res = torch.randn((D, 8), device=dev, generator=g, dtype=torch.float64) / 8
        poles = torch.rand((D, 8), device=dev, generator=g, dtype=torch.float64) * 1.9 - 0.95
        for dt in (torch.float32, torch.bfloat16):
            esz = torch.empty((), dtype=dt).element_size()
            proj = torch.randn((1, 3 * D, L), device=dev, dtype=dt, generator=g)
            feat = torch.randn((3, D, 7), device=dev, generator=g) / 3
            ms = timeit(lambda: ops.li_scan_mixer(proj, feat, res, poles, 1), iters=10)
            report(f"li_scan_mixer_{str(dt)[6:]}", ms, 4 * esz * D * L, D=D, L=L)
            v = proj[:, :D].contiguous()
            ms = timeit(lambda: ops.li_scan(v, res, poles, 1), iters=10)
            report(f"li_scan_ungated_{str(dt)[6:]}", ms, 2 * esz * D * L, D=D, L=L)
            del proj, v
    if args.which in ("all", "kblock"):
        # K-block tcgen05 conv (lh > 129): ungated block_conv, B=4, L=8192, D=4096, bf16
        B, D, L = 4, 4096, 8192
        v = torch.randn((B, D, L), device=dev, dtype=torch.bfloat16, generator=g)
        q = torch.randn_like(v)
        for lh in (200, 300, 513):
            taps = torch.randn((D, lh), device=dev, generator=g) / 20
            ms = timeit(lambda: ops.block_conv(v, taps, 1))
            report(f"block_conv_tcgen05_lh{lh}", ms, 4 * D * B * L, B=B, D=D, L=L, lh=lh)
            ms = timeit(lambda: ops.block_conv(v, taps, 1, q=q, k=q))
            report(f"block_conv_tcgen05_gated_lh{lh}", ms, 8 * D * B * L, B=B, D=D, L=L, lh=lh)
            ms = timeit(lambda: ops.block_conv(v, taps, 16))
            report(f"block_conv_tcgen05_lh{lh}_gs16", ms, 4 * D * B * L, B=B, D=D, L=L, lh=lh, gs=16)
        del v, q
    if args.which in ("all", "qkv"):
        # projection GEMM with the featurizers in its epilogue (tcgen05 CTA pairs) vs cuBLAS on the
        # same W_qkv GEMM, C2 shapes; tensor-bound: reported as TFLOP/s against the measured peak
        B, D, L = 4, 4096, 8192
        x = torch.randn((B, D, L), device=dev, dtype=torch.bfloat16, generator=g)
        w = (torch.randn((3 * D, D), device=dev, generator=g) / 64).to(torch.bfloat16)
        feat = torch.randn((3, D, 7), device=dev, generator=g) / 3
        wp = ops.qkv_weight_permute(w)
        flops = 2.0 * 3 * D * D * B * L
        try:
            peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
        except OSError:
            peak = 1648.3
        for name, fn in (("qkv_feat_gemm", lambda: ops.qkv_feat_gemm(x, wp, feat)),
                         ("cublas_w_qkv_gemm", lambda: torch.matmul(w, x))):
            ms = timeit(fn, iters=10)
            tf = flops / (ms * 1e-3) / 1e12
            print(json.dumps({"kernel": name, "ms": round(ms, 4), "TFLOP/s": round(tf, 1),
                              "frac_bf16_peak": round(tf / peak, 3), "B": B, "D": D, "L": L}), flush=True)
        del x, w, wp
    if args.which in ("all", "fft"):
        D = 4096
        for L, dt in ((131072, torch.bfloat16), (16384, torch.float32)):
            v = torch.randn((1, D, L), device=dev, dtype=dt, generator=g)
            taps = torch.randn((D, L), device=dev, generator=g) / 100
            for path in ("register", "radix4"):
                if path == "radix4":
                    os.environ["HY_FFT_RADIX4"] = "1"
                ms = timeit(lambda: ops.fft_conv(v, taps, 1, q=v, k=v), iters=3, warmup=1)
                os.environ.pop("HY_FFT_RADIX4", None)
                report("fft_conv_" + path, ms, 4 * D * L * v.element_size(), D=D, L=L, dtype=str(dt))
            # cached filter spectra (the operator's path): compute-bound, so also as FP32 TFLOP/s of
            # the two N-point transforms per channel (5 N log2 N each)
            spec = ops.fft_spectrum(taps, L)
            ms = timeit(lambda: ops.fft_conv(v, taps, 1, q=v, k=v, spectrum=spec), iters=3, warmup=1)
            n = 2 * L
            tf = 2 * 5 * n * (n.bit_length() - 1) * D / (ms * 1e-3) / 1e12
            report("fft_conv_spectrum", ms, 4 * D * L * v.element_size(), D=D, L=L, dtype=str(dt),
                   fp32_tflops=round(tf, 1))
            del spec
            del v, taps


if __name__ == "__main__":
    main()
