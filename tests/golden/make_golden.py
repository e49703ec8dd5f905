"""Generate the golden fixtures that pin the oracle to the reference implementation.

Run in the build container, where the reference package is importable (it is not shipped to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything is computed by the reference itself (`gridcast`, float64 numpy) from pinned seeds:
  * neighbor tables (bit-exact, sha256 of little-endian int64) incl. the full-scale (5,90,180)/(5,7,7) table,
    bump_starts cases, the hypothesis-style sweep of test_grid.py:107-120;
  * rotary tables (sha256 of float64 bytes + values for small shapes);
  * init_model_params digests (per-tensor sha256) for tiny / desk / mid configs;
  * natten_block outputs on small shapes, attention weights;
  * tiny and desk forecasts (encode -> rollout -> decode) and the mid-config latent after encode.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("GRIDCAST_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import gridcast.attention as RA  # noqa: E402
import gridcast.grid as RG  # noqa: E402
import gridcast.model as RM  # noqa: E402
import gridcast.rollout as RR  # noqa: E402
from gridcast.autodiff import Tensor, no_grad  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mid_config():
    return RM.ModelConfig(grid=RG.GridSpec(72, 144, lat_step=2.5, lon_step=2.5), surface_in=8, surface_out=17,
                          atmos_vars=5, levels=12, level_patch=2, stem_channels=32, stage_channels=(64, 128, 256),
                          hidden=256, heads=2, window=(5, 7, 7), enc_blocks=2, dec_blocks=2, proc_blocks=10)


def state(cfg, seed):
    rng = np.random.default_rng(seed)
    g = cfg.grid
    return RM.WeatherState(0, rng.standard_normal((cfg.surface_in, g.rows, g.cols)),
                           rng.standard_normal((cfg.atmos_vars, cfg.levels, g.rows, g.cols)))


def main():
    meta: dict = {"neighborhood": [], "bump_starts": [], "rotary": [], "params": {}}
    arrays: dict = {}

    # ---- neighbor tables ----
    cases = [((3, 5, 8), (3, 3, 3)), ((4, 6, 10), (3, 3, 3)), ((1, 5, 6), (1, 3, 1)), ((1, 1, 8), (1, 1, 5)),
             ((7, 9, 18), (5, 7, 7)), ((5, 18, 36), (5, 7, 7)), ((3, 3, 3), (3, 3, 3)), ((2, 7, 10), (1, 4, 4)),
             ((3, 5, 10), (2, 2, 2)), ((5, 90, 180), (5, 7, 7))]
    rng = np.random.default_rng(1234)
    for _ in range(40):  # sweep incl. even windows (test_grid.py:107-120)
        d, h, w = int(rng.integers(1, 7)), int(rng.integers(2, 9)), int(rng.integers(2, 11))
        win = (int(rng.integers(1, d + 1)), int(rng.integers(1, h + 1)), int(rng.integers(1, w + 1)))
        cases.append(((d, h, w), win))
    for ext, win in cases:
        tab = RG.neighborhood(ext, win)
        meta["neighborhood"].append({"extents": ext, "window": win, "sha256": sha(tab.astype("<i8")),
                                     "row0": tab[0, :16].tolist(), "shape": list(tab.shape)})
    for e, w in [(7, 3), (5, 5), (90, 7), (8, 4), (9, 2), (3, 1)]:
        meta["bump_starts"].append({"extent": e, "window": w, "starts": RG.bump_starts(e, w).tolist()})

    # ---- rotary tables ----
    for ext, dh in [((2, 7, 10), 6), ((3, 5, 10), 12), ((7, 9, 18), 128), ((5, 90, 180), 128), ((1, 1, 16), 6)]:
        c, s = RA.rotary_tables(ext, dh)
        meta["rotary"].append({"extents": ext, "head_dim": dh, "cos_sha256": sha(c), "sin_sha256": sha(s)})
        if np.prod(ext) * dh < 5000:
            arrays[f"rot_cos_{'x'.join(map(str, ext))}_{dh}"] = c
            arrays[f"rot_sin_{'x'.join(map(str, ext))}_{dh}"] = s

    # ---- parameter init digests ----
    for name, cfg, seed in [("tiny", RM.tiny_config(), 7), ("desk", RM.desk_config(), 0), ("mid", mid_config(), 7)]:
        p = RM.init_model_params(cfg, seed=seed, zero_residual=False)
        meta["params"][name] = {"seed": seed, "names": list(p), "sha256": {k: sha(v.values) for k, v in p.items()}}

    # ---- natten_block on small shapes ----
    blocks = [("b_2x7x10", (2, 7, 10), (1, 3, 3), 24, 4), ("b_desk", (3, 5, 10), (3, 3, 3), 48, 4),
              ("b_even", (4, 6, 10), (2, 4, 4), 64, 2), ("b_mid", (7, 9, 18), (5, 7, 7), 256, 2)]
    meta["blocks"] = []
    for tag, ext, win, dim, heads in blocks:
        p = RA.init_block_params(np.random.default_rng(0), dim, heads, "blk", zero_residual=False)
        x = np.random.default_rng(2).standard_normal((int(np.prod(ext)), dim))
        with no_grad():
            y = RA.natten_block(Tensor(x), p, "blk", ext, win, heads).values
        aw = RA.attention_weights(x, p, "blk", ext, win, heads)
        arrays[f"{tag}_y"] = y.astype(np.float32) if dim >= 256 else y
        if dim < 256:
            arrays[f"{tag}_attn"] = aw
        meta["blocks"].append({"tag": tag, "extents": ext, "window": win, "dim": dim, "heads": heads,
                               "param_seed": 0, "x_seed": 2})

    # ---- full forecasts ----
    meta["forecasts"] = []
    for tag, cfg, pseed, sseed, dt in [("tiny", RM.tiny_config(), 21, 4, 7), ("desk", RM.desk_config(), 0, 1, 12)]:
        p = RM.init_model_params(cfg, seed=pseed, zero_residual=False)
        st = state(cfg, sseed)
        with no_grad():
            lat = RM.encode(st, p, cfg)
            out = RR.forecast(st, dt, p, cfg)
        arrays[f"fc_{tag}_latent0"] = lat.tokens.values
        arrays[f"fc_{tag}_surface"] = out.surface.values
        arrays[f"fc_{tag}_atmos"] = out.atmos.values
        meta["forecasts"].append({"tag": tag, "param_seed": pseed, "state_seed": sseed, "dt": dt})
    cfg = mid_config()
    p = RM.init_model_params(cfg, seed=7, zero_residual=False)
    with no_grad():
        lat = RM.encode(state(cfg, 1), p, cfg)
    arrays["mid_latent0"] = lat.tokens.values.astype(np.float32)
    meta["mid_encode"] = {"param_seed": 7, "state_seed": 1}

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"), "and golden.npz with", len(arrays), "arrays")


if __name__ == "__main__":
    main()
