"""Host-side profile of backward.rollout_vjp at full scale (one 6 h step, 10 blocks)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2503_22235_b200.model as M
import paper_2503_22235_b200.backward as B
cfg = M.full_scale_config()
params = M.init_model_params(cfg, seed=0, zero_residual=False)
t = int(np.prod(cfg.latent_extents))
z0 = torch.randn(t, cfg.hidden, device="cuda"); gy = torch.randn(t, cfg.hidden, device="cuda")
B.rollout_vjp(z0, (6,), params, cfg, gy)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); B.rollout_vjp(z0, (6,), params, cfg, gy); print("wall (reference grads)", time.perf_counter() - t0)
B.rollout_vjp(z0, (6,), params, cfg, gy, reference_grads=False); torch.cuda.synchronize()
t0 = time.perf_counter(); B.rollout_vjp(z0, (6,), params, cfg, gy, reference_grads=False); torch.cuda.synchronize()
print("wall (device grads)", time.perf_counter() - t0)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
