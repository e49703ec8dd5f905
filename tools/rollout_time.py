"""Time a full-scale 24-step latent rollout (CUDA-graph replays) — A/B aid (e.g. WM3_PDL=1)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m
import paper_2503_22235_b200.rollout as r
from paper_2503_22235_b200.tensor import Tensor
cfg = m.full_scale_config()
params = m.init_model_params(cfg, seed=0, zero_residual=False)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda")
lat = m.LatentState(Tensor(device=x), 0, cfg.latent_extents)
plan = (6,) * 24
r.rollout(lat, plan, params, cfg)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    out = r.rollout(lat, plan, params, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rollout 24x6h: {dt * 1e3:.1f} ms = {dt * 1e3 / (24 * cfg.proc_blocks):.4f} ms/block "
          f"(PDL {'on' if os.environ.get('WM3_PDL') == '1' else 'off'})")
