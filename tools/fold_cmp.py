"""Folded vs separate LayerNorm: per-variable error vs the oracle (tiny/desk/mid, 6 h) and, at full scale, the
divergence between the 8-band emulated forecast and the single-GPU one (a noise-sensitivity probe)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m
import paper_2503_22235_b200.rollout as r
from oracle import model as om

mode = os.environ.get("WM3_LN_FOLD", "1")


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


for name in ["tiny", "desk", "mid"]:
    cfg = {"tiny": m.tiny_config, "desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=7, zero_residual=False)
    host = {k: v.values for k, v in params.items()}
    rng = np.random.default_rng(3)
    g = cfg.grid
    st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    out = r.forecast(st, 6, params, cfg)
    rs, ra = om.forecast(st.surface, st.atmos, 6, host, cfg)
    v = [rel(out.surface.values[i], rs[i]) for i in range(rs.shape[0])]
    v += [rel(out.atmos.values[a, l], ra[a, l]) for a in range(ra.shape[0]) for l in range(ra.shape[1])]
    lat = m.encode(st, params, cfg).tokens.values
    x = lat
    mu = x.mean(1); sd = x.std(1)
    print(f"fold={mode} {name}: per-variable median {np.median(v):.3e} max {max(v):.3e}; latent |mean|/std "
          f"median {np.median(np.abs(mu) / sd):.3f} max {np.max(np.abs(mu) / sd):.3f}")

from paper_2503_22235_b200.bands import forecast_banded
cfg = m.full_scale_config()
params = m.init_model_params(cfg, seed=0, zero_residual=False)
g = cfg.grid
rng = np.random.default_rng(1)
st = m.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).cuda(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32)).cuda())
lat = m.encode(st, params, cfg).tokens.device
mu = lat.mean(1); sd = lat.std(1)
print(f"fold={mode} full-scale latent |mean|/std median {float((mu.abs() / sd).median()):.3f} max {float((mu.abs() / sd).max()):.3f}")
one = r.forecast(st, 7, params, cfg)
b8 = forecast_banded(st, 7, params, cfg, world=8)
a, b = one.surface.device, b8.surface.device
print(f"fold={mode} full scale 8 bands vs single: surface {float((a - b).norm() / a.norm()):.3e} atmos "
      f"{float((one.atmos.device - b8.atmos.device).norm() / one.atmos.device.norm()):.3e}")
np.save(f"gpurun_out/fc_fold{mode}.npy", one.surface.device.cpu().numpy())
