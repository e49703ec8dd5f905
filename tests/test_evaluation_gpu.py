"""Device verification metrics vs golden values computed by the reference's own
evaluation.py (tests/golden/make_eval_golden.py); plus the reference test_evaluation.py invariants
(Parseval, zero RMSE for equal fields, unbounded blur, error classes)."""

import json
import math
import os

import numpy as np
import pytest

from paper_2503_22235_b200.errors import ConfigError, DataError
from paper_2503_22235_b200.grid import GridSpec, desk_grid

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GRIDS = {
    "small": GridSpec(rows=6, cols=8, lat_step=10.0, lon_step=45.0),
    "odd": GridSpec(rows=5, cols=9, lat_step=10.0, lon_step=40.0),
    "desk": desk_grid(),
    "g90": GridSpec(rows=90, cols=180, north_lat=89.0, lat_step=2.0, lon_step=2.0),
}
GOLD = json.load(open(os.path.join(HERE, "eval_golden.json")))
ARR = np.load(os.path.join(HERE, "eval_golden.npz"))


def ev():
    import paper_2503_22235_b200.evaluation as e
    return e


def fields(name, seed, lead=()):
    g = GRIDS[name]
    return np.random.default_rng(seed).standard_normal(tuple(lead) + (g.rows, g.cols))


def close(a, b, tol=1e-11):
    return abs(a - b) <= tol * max(1.0, abs(b))


def test_latitude_rmse_matches_reference():
    for c in GOLD["rmse"]:
        g = GRIDS[c["grid"]]
        p, q = fields(c["grid"], c["seed_p"], (c["times"],)), fields(c["grid"], c["seed_q"], (c["times"],))
        assert close(ev().latitude_rmse(p, q, g), c["value"]), c
        if c["times"] == 1:
            assert ev().latitude_rmse(p[0], q[0], g) == ev().latitude_rmse(p, q, g)
    f = fields("desk", 1, (2,))
    assert ev().latitude_rmse(f, f, GRIDS["desk"]) == 0.0


def test_latitude_rmse_on_device_float32_fields():
    import torch
    g = GRIDS["g90"]
    p, q = fields("g90", 5, (3,)), fields("g90", 6, (3,))
    want = ev().latitude_rmse(p, q, g)
    got = ev().latitude_rmse(torch.from_numpy(p).float().cuda(), torch.from_numpy(q).float().cuda(), g)
    assert abs(got - want) < 1e-6 * want


def test_zonal_power_matches_reference_and_parseval():
    for name in GRIDS:
        g = GRIDS[name]
        f = fields(name, 7)
        p = ev().zonal_power(f, g)
        np.testing.assert_allclose(p, ARR[f"zonal_{name}"], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(p.sum(axis=1), (f * f).mean(axis=1), rtol=1e-10)


def test_power_and_blur_match_reference():
    for c in GOLD["power"]:
        g = GRIDS[c["grid"]]
        assert close(ev().power_at_wavelength(fields(c["grid"], c["seed"]), g, c["wavelength"]), c["value"], 1e-9)
    for c in GOLD["blur"]:
        g = GRIDS[c["grid"]]
        pred = fields(c["grid"], c["seed_pred"]) * c["scale_pred"]
        got = ev().blur_index(pred, fields(c["grid"], c["seed_truth"]), g, c["wavelength"])
        assert close(got, c["value"], 1e-9), (c, got)
    g = GRIDS["desk"]
    f = fields("desk", 7)
    assert ev().blur_index(np.zeros_like(f), f, g, 5000.0) == ev().BLUR_UNBOUNDED
    assert ev().blur_index(f, np.zeros_like(f), g, 5000.0) == ev().BLUR_UNBOUNDED
    assert close(ev().blur_index(f, f, g, 5000.0), 1.0, 1e-12)


def test_ensemble_curve_matches_reference():
    for c in GOLD["curve"]:
        g = GRIDS[c["grid"]]
        members = fields(c["grid"], c["seed_members"], (c["members"], c["times"]))
        truth = fields(c["grid"], c["seed_truth"], (c["times"],))
        rows = ev().ensemble_curve(members, truth, g, wavelength_km=c["wavelength"])
        assert [r["size"] for r in rows] == [r["size"] for r in c["rows"]]
        for got, want in zip(rows, c["rows"]):
            assert close(got["rmse"], want["rmse"]), (got, want)
            assert close(got["blur"], want["blur"], 1e-9), (got, want)


def test_errors_and_scorecard():
    g = GRIDS["small"]
    with pytest.raises(DataError):
        ev().latitude_rmse(np.zeros((6, 8)), np.zeros((3, 3)), g)
    with pytest.raises(DataError):
        ev().latitude_rmse(np.zeros((2, 6, 8)), np.zeros((3, 6, 8)), g)
    with pytest.raises(ConfigError):
        ev().power_at_wavelength(np.zeros((6, 8)), g, -1.0)
    with pytest.raises(ConfigError):
        ev().subset_sizes(0)
    assert ev().subset_sizes(9) == (1, 2, 4, 8)
    sc = ev().scorecard({"a": 1.0, "b": 0.0 + 2.0}, {"a": 2.0, "b": 2.0})
    assert sc == {"a": -50.0, "b": 0.0}
    assert math.isnan(ev().scorecard({"a": 1.0}, {"a": 0.0})["a"])
    with pytest.raises(DataError):
        ev().scorecard({"a": 1.0}, {"b": 1.0})
