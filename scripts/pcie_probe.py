"""Host <-> device copy bandwidth of this box for the e2e leg's per-step transfers (268 MB each way
at C2): H2D alone, D2H alone, and both directions concurrently on two streams (pinned memory)."""
import json

import torch

n = 4 * 4096 * 8192
xh = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
yh = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


h2d = timed(lambda: xd.copy_(xh, non_blocking=True))
d2h = timed(lambda: yh.copy_(yd, non_blocking=True))
bi = timed(both)
gb = n * 2 / 1e9
print(json.dumps({"bytes_each_way": n * 2, "h2d_ms": h2d, "h2d_GBps": gb / h2d * 1e3, "d2h_ms": d2h,
                  "d2h_GBps": gb / d2h * 1e3, "both_ms": bi, "both_GBps_each": gb / bi * 1e3}))
