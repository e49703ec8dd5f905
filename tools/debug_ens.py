"""Debug: ensemble rollout vs single rollouts (graph / eager)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m
import paper_2503_22235_b200.rollout as r

cfg = m.tiny_config()
params = m.init_model_params(cfg, seed=7, zero_residual=False)
rng = np.random.default_rng(8)
g = cfg.grid
st = m.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                    rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))
members = r.perturbed_members(st, 3, scale=0.05)
lats = [m.encode(s, params, cfg) for s in members]
for plan in [(6,), (1,), (6, 1)]:
    ens = r.rollout_ensemble(lats, plan, params, cfg)
    eag = r.rollout_ensemble(lats, plan, params, cfg, graphs=False)
    for k in range(3):
        one = r.rollout(lats[k], plan, params, cfg)
        one_e = r.rollout(lats[k], plan, params, cfg, graphs=False)
        a, b, c, d = (v.tokens.values for v in (ens[k], eag[k], one, one_e))
        print(plan, k, "ens==one", np.array_equal(a, c), "eag==one_e", np.array_equal(b, d), "one==one_e",
              np.array_equal(c, d), "ens==eag", np.array_equal(a, b), float(np.abs(a - c).max()))
