"""Probe: can a gloo process group all-gather CUDA tensors on this box (the WM3_DIST_BACKEND=gloo path of bench.py --gpus 2 on one GPU)?"""
import torch, torch.distributed as dist, os
dist.init_process_group("gloo")
r = dist.get_rank()
t = torch.full((4,), float(r), device="cuda")
out = [torch.empty_like(t) for _ in range(2)]
try:
    dist.all_gather(out, t); print(r, "all_gather cuda ok", [o.tolist() for o in out])
except Exception as e: print(r, "all_gather cuda FAIL", e)
try:
    if r == 0: dist.send(t, 1)
    else:
        u = torch.empty_like(t); dist.recv(u, 0); print(r, "send/recv cuda ok", u.tolist())
except Exception as e: print(r, "send/recv cuda FAIL", str(e)[:200])
try:
    ops = [dist.P2POp(dist.isend, t, 1 - r), dist.P2POp(dist.irecv, torch.empty_like(t), 1 - r)]
    for q in dist.batch_isend_irecv(ops): q.wait()
    print(r, "batch p2p ok")
except Exception as e: print(r, "batch p2p FAIL", str(e)[:200])
x = torch.tensor([1.0 + r], device="cuda"); dist.all_reduce(x, op=dist.ReduceOp.MAX); print(r, "allreduce", x.item())
dist.barrier(); dist.destroy_process_group()
