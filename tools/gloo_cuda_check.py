"""Does gloo send/recv CUDA tensors here? (tools only)"""
import os
import torch
import torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank()
x = torch.full((4,), float(r), device="cuda")
y = torch.empty(4, device="cuda")
ops = [dist.P2POp(dist.isend, x, 1 - r), dist.P2POp(dist.irecv, y, 1 - r)]
for q in dist.batch_isend_irecv(ops):
    q.wait()
print(r, y.tolist(), flush=True)
dist.destroy_process_group()
