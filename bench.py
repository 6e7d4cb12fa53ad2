"""Benchmark: Hyena-MR operator forward (BASELINE.json configs[1]) on B200.

Default workload (N=1): Hyena-MR operator fwd, filter len 128 (two-stage T0/T1),
B=4, L=8192, D=4096, bf16, random-init weights from make_hyena_config and
synthetic N(0,1) inputs. One step = one operator forward over the batch:

    proj = W_qkv^T x (cuBLAS) -> fused featurizers + gates + tcgen05 two-stage
    conv (hy_hyena_mixer_fwd) -> y = W_out^T mixed (cuBLAS)

N > 1 (torchrun, one rank per GPU): independent replicas, each rank runs the
same B=4 batch (weak scaling, no data-path collective; the context-parallel
layer is benchmarked by --workload cp).

--impl reference times the reference algorithm's CPU implementation (the numpy
oracle restatement, oracle/ref.py: float64, as the reference computes) on the
host, one batch element (8192 tokens, full D=4096 width) per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

WORKLOADS = {
    "mr": dict(variant="MR", B=4, L=8192, D=4096, inner_len=128, block_size=128,
               desc="Hyena-MR operator fwd (filter len 128, blocked T0/T1), B=4, L=8192, D=4096, bf16"),
    "se": dict(variant="SE", B=1, L=4096, D=4096, inner_len=7, block_size=16,
               desc="Hyena-SE operator fwd (filter len 7), B=1, L=4096, D=4096, bf16"),
}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return p, "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region
    (written to a file by nvidia-smi itself, read back after the region)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        import tempfile
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        try:
            with open(self.path) as fh:
                lines = fh.read().splitlines()
            os.unlink(self.path)
        except OSError:
            lines = []
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel: str):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
    except OSError:
        return None
    vals = [v["traffic_bytes"] for k, v in sorted(d.items()) if v.get("kernel") == kernel]
    return vals[-1] if vals else None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def build_config(wl: dict):
    import paper_2503_01868_b200 as hy
    return hy.make_hyena_config(wl["variant"], wl["D"], hy.make_rng(0), seq_len=wl["L"], group_size=1,
                                inner_len=wl["inner_len"], block_size=wl["block_size"])


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2503_01868_b200 as hy

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B, D, L = wl["B"], wl["D"], wl["L"]
    cfg = build_config(wl)
    op = hy.HyenaOperator(cfg, torch.bfloat16)
    gen = torch.Generator(device="cuda").manual_seed(1 + rank)
    x = torch.randn((B, D, L), device="cuda", dtype=torch.bfloat16, generator=gen)
    stream = torch.cuda.current_stream()

    def step(ev=None):
        proj = torch.matmul(op.w_qkv_t, x)
        if ev is not None:
            ev[0].record(stream)
        mixed = op.mixer(proj)
        if ev is not None:
            ev[1].record(stream)
        return torch.matmul(op.w_out_t, mixed)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for i in range(args.steps):
        step(evs[i])
    t1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms_total = t0.elapsed_time(t1)
    mixer_ms = [a.elapsed_time(b) for a, b in evs]
    if ws > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps

    # ---- end to end through the public API: pinned host x -> device -> forward -> host y
    xh = torch.empty((B, D, L), dtype=torch.bfloat16, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty((B, D, L), dtype=torch.bfloat16, pin_memory=True)
    for _ in range(max(1, args.warmup)):
        yh.copy_(op.forward(xh.to("cuda", non_blocking=True)), non_blocking=True)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        yh.copy_(op.forward(xh.to("cuda", non_blocking=True)), non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    tokens_step = B * L * ws
    peaks, peaks_kind = load_peaks()
    mix_ms = statistics.mean(mixer_ms)
    mix_bytes = 8 * D * B * L  # (q, k, v projections in + y out) x 2 B per channel per token
    achieved = mix_bytes / (mix_ms * 1e-3) / 1e9
    op_flops = (8 * D * D + 4 * wl["block_size"] * D) * B * L
    result = {
        "metric": "Hyena-MR operator fwd tokens/s (D=4096, % HBM/TC roofline)",
        "value": tokens_step / (ms_step * 1e-3),
        "unit": "tokens/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic N(0,1) inputs, random-init weights (make_hyena_config seed 0)",
        "config": {"workload": wl["desc"], "global_batch": B * ws, "seq_len": L, "width": D,
                   "filter_len": wl["inner_len"], "group_size": 1,
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single",
                   "l2": "inputs (268 MB) larger than L2 (126 MB); no flush"},
        "e2e": {"value": tokens_step / (e2e_ms / args.steps * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(xh.numel() * xh.element_size()),
                "d2h_bytes_per_step": int(yh.numel() * yh.element_size()),
                "path": "HyenaOperator.forward on pinned host bf16 x; H2D + forward + D2H per step"},
        "roofline": {"kernel": "two_stage_kernel<FEAT> (hy_hyena_mixer_fwd: featurizers + gates + tcgen05 T0/T1)",
                     "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "traffic": ncu_traffic("two_stage_kernel"),
                     "peak_source": peaks_kind,
                     "algorithmic_bytes_per_launch": mix_bytes, "launch_ms": mix_ms},
        "roofline_operator": {"bound": "tensor", "achieved": op_flops / (ms_step * 1e-3) / 1e12 / 1,
                              "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                              "frac": op_flops / (ms_step * 1e-3) / 1e12 / peaks["bf16_tflops"],
                              "flops_per_step": op_flops},
        "phases_ms": {"mixer": mix_ms, "gemms": ms_step - mix_ms},
        "clocks": clocks,
        "gpu_launches": args.steps,  # one hy_hyena_mixer_fwd launch per step (projections are cuBLAS)
    }
    if ws > 1:
        dist.destroy_process_group()
    return result, rank


def run_cpu_baseline(wl, max_seconds=30.0):
    """Oracle (numpy, float64 like the reference) on one batch element of the workload."""
    import oracle
    cfg = oracle.make_hyena_config(wl["variant"], wl["D"], oracle.make_rng(0), seq_len=wl["L"], group_size=1,
                                   inner_len=wl["inner_len"], block_size=wl["block_size"])
    x = oracle.make_rng(1, stream=0).standard_normal((wl["D"], wl["L"]))
    times = []
    start = time.perf_counter()
    while True:
        t = time.perf_counter()
        oracle.hyena_forward(x, cfg)
        times.append(time.perf_counter() - t)
        if time.perf_counter() - start > max_seconds * 0.5 or len(times) >= 3:
            break
    med = statistics.median(times)
    return {"value": wl["L"] / med, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle.hyena_forward (numpy float64 restatement of hyena.py:157-190) on 1 of {wl['B']} "
                      f"batch elements ({wl['L']} tokens, D={wl['D']}), median of {len(times)} calls; "
                      f"OpenBLAS threads = all {os.cpu_count()} host cores"}


def run_reference(args, wl, sample_len=2048):
    """Reference arm: the reference algorithm's CPU implementation (numpy oracle port, float64)
    on the host; each step is one forward over a (D, sample_len) token sample of one batch
    element (per-token cost of the operator is independent of L: projections, featurizer
    and two-stage conv are all linear in L)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return None, rank
    import oracle
    cfg = oracle.make_hyena_config(wl["variant"], wl["D"], oracle.make_rng(0), seq_len=wl["L"], group_size=1,
                                   inner_len=wl["inner_len"], block_size=wl["block_size"])
    x = oracle.make_rng(1, stream=0).standard_normal((wl["D"], wl["L"]))[:, :sample_len].copy()
    for _ in range(args.warmup):
        oracle.hyena_forward(x, cfg)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.hyena_forward(x, cfg)
    ms = (time.perf_counter() - t) * 1e3 / args.steps
    value = sample_len / (ms * 1e-3)
    sample = (f"each step: one forward over {sample_len} of the {wl['L']} tokens of one batch element at full "
              f"D={wl['D']} (numpy float64 oracle port of hyena.py:157-190; OpenBLAS on all host cores)")
    return {
        "impl": "reference", "metric": "Hyena-MR operator fwd tokens/s (D=4096, % HBM/TC roofline)",
        "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic N(0,1) inputs, random-init weights (make_hyena_config seed 0)",
        "config": {"workload": wl["desc"], "global_batch": wl["B"], "seq_len": wl["L"], "width": wl["D"]},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }, rank


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="mr", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        res, rank = run_reference(args, wl)
    else:
        res, rank = run_ours(args, wl)
        if rank == 0 and res["n_gpus"] == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = run_cpu_baseline(wl)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
