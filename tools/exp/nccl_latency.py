"""Latency of the per-step winner exchange (all_gather of 40 bytes) on N GPUs:
torchrun --nproc-per-node N tools/exp/nccl_latency.py"""
import os
import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
x = torch.zeros(40, dtype=torch.uint8, device="cuda")
out = torch.empty(40 * dist.get_world_size(), dtype=torch.uint8, device="cuda")
for _ in range(20):
    dist.all_gather_into_tensor(out, x)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(200):
    dist.all_gather_into_tensor(out, x)
b.record()
torch.cuda.synchronize()
if r == 0:
    print(f"all_gather 40 B x {dist.get_world_size()}: {a.elapsed_time(b) / 200 * 1e3:.1f} us per call")
dist.destroy_process_group()
