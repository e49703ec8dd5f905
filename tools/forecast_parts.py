"""Time the parts of a full-scale forecast: host->device + encode, one 6 h processor step, decode + device->host."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m
import paper_2503_22235_b200.rollout as r
cfg = m.full_scale_config()
params = m.init_model_params(cfg, seed=0, zero_residual=False)
g = cfg.grid
rng = np.random.default_rng(1)
st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32),
                    rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32))


def t(fn, n=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, out


te, lat = t(lambda: m.encode(st, params, cfg))
tp, lat6 = t(lambda: r.rollout(lat, (6,), params, cfg, graphs=False))
td, dec = t(lambda: m.decode(lat6, params, cfg))
th, _ = t(lambda: (dec.surface.device.cpu(), dec.atmos.device.cpu()))
print(f"encode {te*1e3:.1f} ms (21.58 TF convs + 2 blocks) | process6 {tp*1e3:.1f} ms | decode {td*1e3:.1f} ms "
      f"(31.31 TF convs + 2 blocks) | D2H fields {th*1e3:.1f} ms")
