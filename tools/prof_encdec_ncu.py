"""One warm-up full-scale encode + decode, then a second one for ncu to capture (profiles/r2_encdec.md):
    ncu --set full -k regex:"conv_tc|fields_to_nhwc|tokens_to_nhwc" -s 37 -c 37 python tools/prof_encdec_ncu.py
(37 = 2 fields_to_nhwc + 17 convs per encode, 1 tokens_to_nhwc + 17 convs per decode; the round-2 capture used
-s 39 and so starts at the atmosphere fields_to_nhwc of the second pass)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_22235_b200.model as m  # noqa: E402

cfg = m.full_scale_config()
params = m.init_model_params(cfg, seed=0, zero_residual=False)
g = cfg.grid
rng = np.random.default_rng(1)
st = m.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, g.rows, g.cols)).astype(np.float32)).cuda(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols))
                                     .astype(np.float32)).cuda())
for _ in range(2):
    lat = m.encode(st, params, cfg)
    dec = m.decode(lat, params, cfg)
    torch.cuda.synchronize()
print("ok", float(dec.surface.device.abs().mean()))
