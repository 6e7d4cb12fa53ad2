"""Times the C3 LI operator through the default route (cuBLAS W_qkv + fused LI mixer) and the fused
projection route (hy_qkv_feat_gemm + li_conv gated by fq), and the two routes' parts; one JSON line."""
import json, os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_2503_01868_b200 as hy
import bench
wl = bench.WORKLOADS["li"]
cfg = bench.build_config(wl)
op = hy.HyenaOperator(cfg, torch.bfloat16)
x = torch.randn((1, 4096, 131072), device="cuda").to(torch.bfloat16)
def timed(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
out = {}
for rep in range(2):
    op.qkv_fused = False
    out[f"default_{rep}"] = timed(lambda: op.forward(x))
    op.qkv_fused = True
    out[f"fused_{rep}"] = timed(lambda: op.forward(x))
fq, u = op.project_featurized(x)
out["li_conv_gated_ms"] = timed(lambda: op.inner_gated(u, fq))
proj = op.project(x)
out["li_mixer_ms"] = timed(lambda: op.mixer(proj))
out["cublas_proj_ms"] = timed(lambda: op.project(x))
out["fused_proj_ms"] = timed(lambda: op.project_featurized(x))
print(json.dumps(out))
