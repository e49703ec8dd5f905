"""Timeline of config 3's encode and decode with page-locked host fields (torch.profiler / CUPTI): when the host
copies run, when the kernels run, and how much of each is exposed (not overlapped by the other)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as M
from torch.profiler import ProfilerActivity, profile

cfg = M.full_scale_config()
params = M.init_model_params(cfg, seed=0, zero_residual=False)
g = cfg.grid
rng = np.random.default_rng(1)
st = M.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).pin_memory(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols))
                                     .astype(np.float32)).pin_memory())
lat = M.encode(st, params, cfg)
dec = M.decode(lat, params, cfg)
host = dec.to_host()
torch.cuda.synchronize()


def intervals(evs):
    out = []
    for e in evs:
        s = e.time_range.start if hasattr(e, "time_range") else e.start_us()
        out.append((e.time_range.start, e.time_range.end, e.name))
    return sorted(out)


def union(iv):
    tot, cur = 0.0, None
    for s, e, _ in sorted(iv):
        if cur is None or s > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [s, e]
        else:
            cur[1] = max(cur[1], e)
    if cur:
        tot += cur[1] - cur[0]
    return tot


lat6 = M.process(lat, params, cfg, 6)
torch.cuda.synchronize()
for name, fn in (("encode", lambda: M.encode(st, params, cfg)), ("process6", lambda: M.process(lat, params, cfg, 6)),
                 ("decode", lambda: M.decode(lat6, params, cfg, host_out=host).to_host(host))):
    fn()  # steady state: the previous call's outputs released, caches warm
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    cp = [(e.time_range.start, e.time_range.end, e.name) for e in evs if "emcpy" in e.name or "Memcpy" in e.name]
    kn = [(e.time_range.start, e.time_range.end, e.name) for e in evs if not ("emcpy" in e.name or "Memcpy" in e.name)]
    t0 = min(s for s, _, _ in cp + kn)
    t1 = max(e for _, e, _ in cp + kn)
    both = union(cp + kn)
    print(f"{name}: span {(t1 - t0) / 1e3:.2f} ms, copies {union(cp) / 1e3:.2f} ms ({len(cp)}), kernels "
          f"{union(kn) / 1e3:.2f} ms ({len(kn)}), busy {both / 1e3:.2f} ms, copy-only {(both - union(kn)) / 1e3:.2f} ms, "
          f"kernel-only {(both - union(cp)) / 1e3:.2f} ms, idle {(t1 - t0 - both) / 1e3:.2f} ms")
    allv = sorted(cp + kn)
    gaps, end, prev = [], None, None
    for s_, e_, n_ in allv:
        if end is not None and s_ > end:
            gaps.append((s_ - end, end, prev, n_))
        if end is None or e_ > end:
            end, prev = e_, n_
    for d_, at, a, b in sorted(gaps, reverse=True)[:4]:
        print(f"   idle {d_ / 1e3:6.3f} ms at {(at - t0) / 1e3:7.2f} ms: after {a[:40]} | before {b[:40]}")

