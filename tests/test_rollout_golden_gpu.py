"""Long-rollout parity against fixtures produced by the reference itself (tests/golden/make_rollout_golden.py):
BASELINE config 4 (24 h greedy rollout (6, 6, 6, 6) and (6, 1), latent space, mid config with the paper's
(5, 7, 7) window) and config 5's 14-day horizon (greedy_plan(336) = 56 six-hour steps, decoded fields per
variable) on the desk and mid configs.  Tolerance: full rollout, latent and
per-variable relative L2 <= 2e-2."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixtures():
    with open(os.path.join(HERE, "rollout_golden.json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(HERE, "rollout_golden.npz"))


def _setup(name, meta):
    import paper_2503_22235_b200.model as m
    cfg = {"desk": m.desk_config, "mid": m.mid_config}[name]()
    params = m.init_model_params(cfg, seed=meta["param_seed"], zero_residual=False)
    rng = np.random.default_rng(meta["state_seed"])
    g = cfg.grid
    st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
    return cfg, params, st


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("tag,dt", [("mid_24h", 24), ("mid_7h", 7)])
def test_mixed_horizon_rollout_latent_vs_reference(tag, dt):
    import paper_2503_22235_b200.model as m
    import paper_2503_22235_b200.rollout as r
    meta, arrs = _fixtures()
    cfg, params, st = _setup("mid", meta)
    lat = m.encode(st, params, cfg)
    out = r.rollout(lat, r.greedy_plan(dt), params, cfg)
    assert out.valid_time == dt
    rel = _rel(out.tokens.values, arrs[f"{tag}_latent"].astype(np.float64))
    print(f"[{tag}] latent rel L2 {rel:.3e}")
    assert rel < 2e-2, rel


@pytest.mark.parametrize("name", ["desk", "mid"])
def test_fourteen_day_forecast_per_variable_vs_reference(name):
    import paper_2503_22235_b200.rollout as r
    meta, arrs = _fixtures()
    cfg, params, st = _setup(name, meta)
    out = r.forecast(st, 336, params, cfg)
    assert out.valid_time == 336
    ref_s, ref_a = arrs[f"{name}_336h_surface"], arrs[f"{name}_336h_atmos"]
    got_s, got_a = out.surface.values, out.atmos.values
    rel = {f"sfc{i}": _rel(got_s[i], ref_s[i]) for i in range(ref_s.shape[0])}
    rel.update({f"atm{a}.lev{lev}": _rel(got_a[a, lev], ref_a[a, lev])
                for a in range(ref_a.shape[0]) for lev in range(ref_a.shape[1])})
    worst = max(rel, key=rel.get)
    vals = np.array(sorted(rel.values()))
    print(f"[{name} 336 h] per-variable rel L2: median {np.median(vals):.2e} max {vals[-1]:.2e} ({worst})")
    assert rel[worst] < 2e-2, (worst, rel[worst])
