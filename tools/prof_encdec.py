"""Per-kernel device times of one full-scale encode and decode (torch.profiler / CUPTI)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m
cfg = m.full_scale_config()
params = m.init_model_params(cfg, seed=0, zero_residual=False)
g = cfg.grid
rng = np.random.default_rng(1)
st = m.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).cuda(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)).astype(np.float32)).cuda())
lat = m.encode(st, params, cfg)
dec = m.decode(lat, params, cfg)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
for name, fn in [("encode", lambda: m.encode(st, params, cfg)), ("decode", lambda: m.decode(lat, params, cfg))]:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    tot = sum(e.device_time for e in evs)
    print(f"== {name}: {len(evs)} kernels, {tot / 1e3:.2f} ms device time")
    for e in evs:
        print(f"   {e.device_time / 1e3:8.3f} ms  {e.name[:90]}")
