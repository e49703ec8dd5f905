"""Idle gaps of the GPU during a full-scale 14-day forecast with page-locked host fields (torch.profiler / CUPTI):
host-side stalls between the encode, the rollout's graph replays and the decode show up as idle time."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as M
import paper_2503_22235_b200.rollout as R
from torch.profiler import ProfilerActivity, profile

cfg = M.full_scale_config()
params = M.init_model_params(cfg, seed=0, zero_residual=False)
g = cfg.grid
rng = np.random.default_rng(1)
st = M.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).pin_memory(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols))
                                     .astype(np.float32)).pin_memory())
dt = int(sys.argv[1]) if len(sys.argv) > 1 else 336
out = R.forecast(st, dt, params, cfg)
host = out.to_host()
torch.cuda.synchronize()
R.forecast(st, dt, params, cfg, host_out=host).to_host(host)
torch.cuda.synchronize()
t0w = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    R.forecast(st, dt, params, cfg, host_out=host).to_host(host)
    torch.cuda.synchronize()
wall = time.perf_counter() - t0w
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events() if e.device_type.name == "CUDA")
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
gaps, end, prev = [], None, None
busy = 0.0
for s_, e_, n_ in iv:
    if end is not None and s_ > end:
        gaps.append((s_ - end, end, prev, n_))
    if end is None or e_ > end:
        busy += e_ - max(s_, end if end is not None else s_)
        end, prev = e_, n_
print(f"forecast {dt} h: wall {wall * 1e3:.1f} ms (under profiler), device span {(t1 - t0) / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, "
      f"idle {sum(g_[0] for g_ in gaps) / 1e3:.2f} ms in {len(gaps)} gaps")
for d_, at, a, b in sorted(gaps, reverse=True)[:10]:
    print(f"   idle {d_ / 1e3:6.3f} ms at {(at - t0) / 1e3:8.2f} ms: after {a[:40]} | before {b[:40]}")
