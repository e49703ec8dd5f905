"""Long-rollout fixtures from the reference itself (BASELINE configs 4 and 5 at oracle-feasible scale).

Run in the build container, where the reference package is importable (it is not shipped to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_rollout_golden.py

Writes tests/golden/rollout_golden.{json,npz}, all computed by `gridcast` (float64 numpy), stored as float32:
  * mid config: the latent after the 24 h greedy rollout (6, 6, 6, 6) and after (6, 1) from encode(state);
  * desk config: the full 14-day forecast (greedy_plan(336) = 56 six-hour steps) decoded fields;
  * mid config: the full 14-day forecast decoded fields (56 x 10 processor blocks on the paper's window).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("GRIDCAST_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import gridcast.model as RM  # noqa: E402
import gridcast.rollout as RR  # noqa: E402
from gridcast.autodiff import no_grad  # noqa: E402
from make_golden import mid_config, state  # noqa: E402


def main():
    arrays, meta = {}, {"param_seed": 7, "state_seed": 4, "runs": []}
    t0 = time.time()
    cfg = mid_config()
    p = RM.init_model_params(cfg, seed=7, zero_residual=False)
    with no_grad():
        lat = RM.encode(state(cfg, 4), p, cfg)
        for tag, dt in (("mid_24h", 24), ("mid_7h", 7)):
            out = RR.rollout(lat, RR.greedy_plan(dt), p, cfg)
            arrays[f"{tag}_latent"] = out.tokens.values.astype(np.float32)
            meta["runs"].append({"tag": tag, "config": "mid", "dt": dt, "plan": list(RR.greedy_plan(dt)),
                                 "kind": "latent"})
            print(tag, f"{time.time() - t0:.1f}s", flush=True)
    for tag, cfg_name in (("desk_336h", "desk"), ("mid_336h", "mid")):
        cfg = RM.desk_config() if cfg_name == "desk" else mid_config()
        p = RM.init_model_params(cfg, seed=7, zero_residual=False)
        with no_grad():
            out = RR.forecast(state(cfg, 4), 336, p, cfg)
        arrays[f"{tag}_surface"] = out.surface.values.astype(np.float32)
        arrays[f"{tag}_atmos"] = out.atmos.values.astype(np.float32)
        meta["runs"].append({"tag": tag, "config": cfg_name, "dt": 336, "kind": "fields"})
        print(tag, f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(HERE, "rollout_golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "rollout_golden.npz"), **arrays)
    print("wrote rollout_golden.{json,npz} with", len(arrays), "arrays", f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
