"""Full-scale reverse mode: one block VJP (device, per phase) and a one-step (10-block) rollout VJP with and
without host offload, CUDA-event timed."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as M
from paper_2503_22235_b200.backward import BlockGrads, block_vjp_device, rollout_vjp
from paper_2503_22235_b200.runtime import CACHE

cfg = M.full_scale_config()
params = M.init_model_params(cfg, seed=0, zero_residual=False)
ext, win, heads, dh = cfg.latent_extents, cfg.window, cfg.heads, cfg.head_dim
t = int(np.prod(ext))
x = torch.randn(t, cfg.hidden, device="cuda")
gy = torch.randn(t, cfg.hidden, device="cuda")
bw = CACHE.block(params, "proc6.blk0", heads)
for _ in range(2):
    block_vjp_device(x, bw, ext, win, heads, dh, gy, BlockGrads())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    block_vjp_device(x, bw, ext, win, heads, dh, gy, BlockGrads())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"block VJP (recompute + backward) full scale: {ms:.2f} ms = {3 * 2.1197e12 / (ms / 1e3) / 1e12:.0f} TFLOP/s "
      f"(3x the forward's algorithmic FLOPs)")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    block_vjp_device(x, bw, ext, win, heads, dh, gy, BlockGrads())
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.split("(")[0][:60]
        agg[k] = agg.get(k, 0.0) + e.device_time / 1e3
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
    print(f"   {v:8.3f} ms  {k}")
z0 = torch.randn(t, cfg.hidden, device="cuda")
for off in (False, True):
    rollout_vjp(z0, (6,), params, cfg, gy, offload=off)
    t0 = time.perf_counter()
    _, _, _, st = rollout_vjp(z0, (6,), params, cfg, gy, offload=off)
    print(f"rollout_vjp (6,) offload={off}: {time.perf_counter() - t0:.3f} s wall incl. host gradient copies, {st}")
