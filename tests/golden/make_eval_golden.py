"""Golden vectors for the verification metrics, computed by the reference itself (run in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_eval_golden.py

Inputs are regenerated in the tests from the recorded seeds (numpy default_rng), so only outputs are stored:
tests/golden/eval_golden.npz (zonal power spectra) and tests/golden/eval_golden.json (scalars and curves).
"""
import json
import os

import numpy as np

from gridcast.evaluation import blur_index, ensemble_curve, latitude_rmse, power_at_wavelength, zonal_power
from gridcast.grid import GridSpec, desk_grid

HERE = os.path.dirname(os.path.abspath(__file__))
GRIDS = {
    "small": GridSpec(rows=6, cols=8, lat_step=10.0, lon_step=45.0),
    "odd": GridSpec(rows=5, cols=9, lat_step=10.0, lon_step=40.0),
    "desk": desk_grid(),
    "g90": GridSpec(rows=90, cols=180, north_lat=89.0, lat_step=2.0, lon_step=2.0),
}


def fields(name, seed, lead=()):
    g = GRIDS[name]
    return np.random.default_rng(seed).standard_normal(tuple(lead) + (g.rows, g.cols))


def run():
    js, arrays = {"rmse": [], "power": [], "blur": [], "curve": []}, {}
    for name in GRIDS:
        g = GRIDS[name]
        for t in (1, 3):
            p, q = fields(name, 100 + t, (t,)), fields(name, 200 + t, (t,))
            js["rmse"].append({"grid": name, "times": t, "seed_p": 100 + t, "seed_q": 200 + t,
                               "value": latitude_rmse(p, q, g)})
        f = fields(name, 7)
        arrays[f"zonal_{name}"] = zonal_power(f, g)
    for name, wls in [("desk", [2000.0, 5000.0, 12000.0]), ("g90", [1000.0, 3000.0, 8000.0])]:
        g = GRIDS[name]
        f, h = fields(name, 7), fields(name, 8) * 0.7
        for wl in wls:
            js["power"].append({"grid": name, "seed": 7, "wavelength": wl, "value": power_at_wavelength(f, g, wl)})
            js["blur"].append({"grid": name, "seed_pred": 8, "scale_pred": 0.7, "seed_truth": 7, "wavelength": wl,
                               "value": blur_index(h, f, g, wl)})
    for name, n, t, wl in [("desk", 5, 2, 5000.0), ("g90", 9, 1, 3000.0)]:
        g = GRIDS[name]
        members, truth = fields(name, 300, (n, t)), fields(name, 301, (t,))
        js["curve"].append({"grid": name, "members": n, "times": t, "seed_members": 300, "seed_truth": 301,
                            "wavelength": wl, "rows": ensemble_curve(members, truth, g, wavelength_km=wl)})
    np.savez(os.path.join(HERE, "eval_golden.npz"), **arrays)
    with open(os.path.join(HERE, "eval_golden.json"), "w") as fh:
        json.dump(js, fh, indent=1)


if __name__ == "__main__":
    run()
