"""Smoke test of p2p.PeerAllToAll under torchrun: exchange, compare with all_to_all_single."""
import os, sys, torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_01868_b200.p2p import PeerAllToAll
r = int(os.environ["RANK"]); n = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(r)
dist.init_process_group("nccl", rank=r, world_size=n, device_id=torch.device("cuda", r))
ex = PeerAllToAll(dist.group.WORLD, (64, 4096), torch.bfloat16)
ok = True
for it in range(6):
    send = torch.randn((n, 64, 4096), device="cuda").to(torch.bfloat16) + it
    ref = torch.empty_like(send)
    dist.all_to_all_single(ref, send)
    k = it % 2
    got = ex.exchange(send, k).clone()
    ex.release(k)
    torch.cuda.synchronize()
    ok &= torch.equal(got, ref)
print(f"rank {r}: p2p all-to-all matches NCCL: {ok}", flush=True)
dist.destroy_process_group()
