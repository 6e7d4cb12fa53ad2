cat > /tmp/mix_t.py <<'PY'
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2503_01868_b200 import ops
def timed(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record(); torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 4)
D = 4096
g = torch.Generator(device="cuda").manual_seed(0)
feat = torch.randn((3, D, 7), device="cuda", generator=g) / 3
packed = ops.feat_pack(feat)
taps = torch.randn((D, 128), device="cuda", generator=g) / 11
res = torch.randn((D, 8), device="cuda", generator=g) / 8
poles = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
out = {"lib": os.environ["LIB"]}
proj = torch.randn((4, 3 * D, 8192), device="cuda", generator=g).to(torch.bfloat16)
out["mr_C2"] = timed(lambda: ops.hyena_mixer(proj, feat, taps, 1, packed=packed))
del proj
for L in (16384, 131072):
    proj = torch.randn((1, 3 * D, L), device="cuda", generator=g).to(torch.bfloat16)
    out[f"li_L{L}"] = timed(lambda: ops.li_mixer(proj, feat, res, poles, 1, packed=packed), reps=10)
    del proj
print(json.dumps(out))
PY
for v in old new old new; do cp ab_libs/$v.so paper_2503_01868_b200/libhyena_b200.so; LIB=$v timeout 200 python /tmp/mix_t.py; done
cp ab_libs/new.so paper_2503_01868_b200/libhyena_b200.so
