"""Per-kernel CUDA time of one context-parallel LI forward step (torch profiler), rank 0."""
import os, sys, torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_01868_b200 import cp
ws = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(rank)
dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", rank))
wl = bench.WORKLOADS["li_cp"]
mod = cp.HyenaCP(bench.build_config(wl), torch.bfloat16)
m = wl["L"] // ws
x = torch.randn((1, wl["D"], m), device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    mod.forward(x)
torch.cuda.synchronize(); dist.barrier()
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    mod.forward(x)
    torch.cuda.synchronize()
if rank == 0:
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18, max_name_column_width=70))
dist.destroy_process_group()
