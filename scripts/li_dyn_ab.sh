# dynamic vs static IMPL scheduling (and the pre-change library): LI mixer timings + SM clock
mkdir -p gpurun_out
cat > /tmp/li_t.py <<'PY'
import json, os, sys, torch
sys.path.insert(0, '.')
from paper_2503_01868_b200 import ops
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
def timed(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): f()
    e.record()
    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    torch.cuda.synchronize()
    return round(s.elapsed_time(e) / reps, 4), mhz
D = 4096
out = {"lib": os.environ.get("LIB"), "dyn": os.environ.get("HY_LI_DYNAMIC", "1")}
g = torch.Generator(device="cuda").manual_seed(0)
res = torch.randn((D, 8), device="cuda", generator=g) / 8
poles = torch.rand((D, 8), device="cuda", generator=g) * 1.9 - 0.95
feat = torch.randn((3, D, 7), device="cuda", generator=g) / 3
packed = ops.feat_pack(feat)
for L in (16384, 131072):
    proj = torch.randn((1, 3 * D, L), device="cuda", generator=g).to(torch.bfloat16)
    out[f"li_mixer_L{L}"] = timed(lambda: ops.li_mixer(proj, feat, res, poles, 1, packed=packed))
    del proj
taps = torch.randn((D, 128), device="cuda", generator=g) / 11
proj = torch.randn((4, 3 * D, 8192), device="cuda", generator=g).to(torch.bfloat16)
out["mr_mixer_C2"] = timed(lambda: ops.hyena_mixer(proj, feat, taps, 1, packed=packed))
print(json.dumps(out))
PY
for v in old:0 v1:0 v2:0 new:0 old:0 v1:0 v2:0; do
  lib=${v%%:*}; d=${v##*:}
  cp ab_libs/$lib.so paper_2503_01868_b200/libhyena_b200.so
  LIB=$lib HY_LI_DYNAMIC=$d timeout 300 python /tmp/li_t.py
done
