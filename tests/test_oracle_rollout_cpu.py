"""The oracle pinned to the reference's long rollouts (tests/golden/rollout_golden.*, written by the reference
itself via make_rollout_golden.py; stored float32, so agreement is to float32 rounding): the mid-config 24 h
greedy rollout (6, 6, 6, 6) in latent space and the desk-config 14-day forecast (56 six-hour steps)."""

import json
import os

import numpy as np

from oracle import model as om

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
META = json.load(open(os.path.join(HERE, "rollout_golden.json")))
ARR = np.load(os.path.join(HERE, "rollout_golden.npz"))


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _inputs(cfg):
    from paper_2503_22235_b200.params import init_model_params
    p = {k: v.values for k, v in init_model_params(cfg, seed=META["param_seed"], zero_residual=False).items()}
    rng = np.random.default_rng(META["state_seed"])
    g = cfg.grid
    return p, rng.standard_normal((cfg.surface_in, g.rows, g.cols)), \
        rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols))


def test_oracle_mid_24h_rollout_matches_reference():
    from paper_2503_22235_b200 import config as C
    cfg = C.mid_config()
    p, sfc, atm = _inputs(cfg)
    lat = om.rollout(om.encode(sfc, atm, p, cfg), om.greedy_plan(24), p, cfg)
    assert _rel(lat, ARR["mid_24h_latent"].astype(np.float64)) < 1e-6


def test_oracle_desk_14_day_forecast_matches_reference():
    from paper_2503_22235_b200 import config as C
    cfg = C.desk_config()
    p, sfc, atm = _inputs(cfg)
    s, a = om.forecast(sfc, atm, 336, p, cfg)
    assert _rel(s, ARR["desk_336h_surface"].astype(np.float64)) < 1e-6
    assert _rel(a, ARR["desk_336h_atmos"].astype(np.float64)) < 1e-6
