"""Times the fused projection GEMM (hy_qkv_feat_gemm) against cuBLAS's W_qkv GEMM at C2 size
(B = 4, D = 4096, L = 8192), and the two MR mixer routes: cuBLAS GEMM + the fused FEAT mixer vs
the fused GEMM + the K-block conv on [fq; u]. One JSON line per measurement."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200 import ops  # noqa: E402


try:
    import pynvml
    pynvml.nvmlInit()
    _NV = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # clocks are informational
    _NV = None
CLOCKS = {}


def timed(fn, reps=20, warm=3, name=None):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    if _NV is not None and name:  # SM clock while the queued launches run
        CLOCKS[name] = pynvml.nvmlDeviceGetClockInfo(_NV, pynvml.NVML_CLOCK_SM)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    B, D, L = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4, 4096, 8192)))
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((B, D, L), device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn((3 * D, D), device="cuda", generator=g) / D ** 0.5).to(torch.bfloat16)
    feat = torch.randn((3, D, 7), device="cuda", generator=g) / 2.65
    taps = torch.randn((D, 128), device="cuda", generator=g) / 11.3
    dec = torch.linspace(0.01, 2.0, D, device="cuda")
    wp = ops.qkv_weight_permute(w)
    packed = ops.feat_pack(feat)
    flops = 2.0 * 3 * D * D * B * L
    out = {}
    for rep in range(3):  # interleaved: power / clock state affects both alike
        out[f"cublas_gemm_ms_{rep}"] = timed(lambda: torch.matmul(w, x), reps=40, name=f"cublas_{rep}")
        out[f"fused_gemm_ms_{rep}"] = timed(lambda: ops.qkv_feat_gemm(x, wp, feat), reps=40, name=f"fused_{rep}")
    out["cublas_gemm_ms"] = min(out[f"cublas_gemm_ms_{r}"] for r in range(3))
    out["fused_gemm_ms_s0"] = min(out[f"fused_gemm_ms_{r}"] for r in range(3))
    for s in [int(v) for v in os.environ.get("QG_SEGMENTS", "").split(",") if v]:
        out[f"fused_gemm_ms_s{s}"] = timed(lambda: ops.qkv_feat_gemm(x, wp, feat, segments=s))
    out["fused_gemm_tflops"] = flops / out["fused_gemm_ms_s0"] / 1e9
    out["cublas_gemm_tflops"] = flops / out["cublas_gemm_ms"] / 1e9
    proj = torch.matmul(w, x)
    out["feat_mixer_ms"] = timed(lambda: ops.hyena_mixer(proj, feat, taps, 1, decay=dec, packed=packed))
    fq, u = ops.qkv_feat_gemm(x, wp, feat)
    out["block_conv_fq_u_ms"] = timed(lambda: ops.block_conv(u, taps, 1, q=fq, decay=dec))
    out["block_conv_fq_u_nodecay_ms"] = timed(lambda: ops.block_conv(u, taps, 1, q=fq))
    out["two_stage_fq_u_ms"] = timed(lambda: ops.two_stage(u, taps, 1, q=fq, decay=dec))
    out["route_cublas_plus_mixer_ms"] = timed(
        lambda: ops.hyena_mixer(torch.matmul(w, x), feat, taps, 1, decay=dec, packed=packed))
    out["route_fused_plus_block_conv_ms"] = timed(
        lambda: (lambda f: ops.block_conv(f[1], taps, 1, q=f[0], decay=dec))(ops.qkv_feat_gemm(x, wp, feat)))
    out.update(B=B, D=D, L=L, gpu=torch.cuda.get_device_name(), sm_mhz=CLOCKS)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
