"""Summarise ncu captures into profiles/ (run here, after gpurun brought the .ncu-rep back).

    python scripts/ncu_summary.py gpurun_out/prof_mr.ncu-rep profiles/r01_mr_mixer_ncu.txt mr
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv profiles/r01_launches.txt
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__block_size",
    "launch__grid_size",
    "sm__cycles_elapsed.avg.per_second",
]


def raw_metrics(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    res = {"kernel": name}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            res[k] = f"{vals[i]} {units[i]}".strip()
    return res


def summarize_rep(rep: str, dst: str, workload: str | None = None) -> None:
    m = raw_metrics(rep)
    lines = [f"ncu --set full capture: {os.path.basename(rep)}", f"kernel: {m.pop('kernel')}", ""]
    lines += [f"{k:85s} {v}" for k, v in m.items()]
    scales = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def nbytes(key):  # each metric carries its own unit
        val, unit = m[key].split()[:2]
        return float(val.replace(",", "")) * scales[unit]

    traffic = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    lines += ["", f"traffic (dram read + write) per launch: {traffic:.0f} bytes"]
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tj = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    ent = {"kernel": lines[1][len("kernel: "):], "traffic_bytes": traffic}
    if workload:
        ent["workload"] = workload
    d[os.path.basename(dst)] = ent
    json.dump(d, open(tj, "w"), indent=1)


def summarize_launches(src: str, dst: str) -> None:
    rows = list(csv.reader(open(src)))
    i = [k for k, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[i + 1:]:
        if len(r) > vi:
            d[r[ki]].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in d.values())
    lines = [f"ncu launch list (gpu__time_duration.sum, --clock-control none, cold-cache serialised): {src}",
             f"{'launches':>8} {'avg_us':>10} {'share':>7}  kernel"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / total:7.1%}  {k[:110]}")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        summarize_launches(sys.argv[2], sys.argv[3])
    else:
        summarize_rep(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
