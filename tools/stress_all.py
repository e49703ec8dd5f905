"""Bitwise-repeatability stress beyond the GEMMs: the NA kernel, the full block, the encoder / decoder pyramids
and the LayerNorm, each run N times on identical inputs (any mismatch = a race)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_22235_b200 import _lib as L, ops
from paper_2503_22235_b200.blocks import RopeTables, Workspace, block_forward, prepare_block
from paper_2503_22235_b200.params import init_block_params
import paper_2503_22235_b200.model as m

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
ext, win, dim, heads = (5, 90, 180), (5, 7, 7), 1024, 8
t = 81000
g = torch.Generator(device="cuda").manual_seed(0)
bad = {}


def stress(name, f, n=N):
    ref = [r.clone() for r in f()]
    torch.cuda.synchronize()
    k = 0
    for _ in range(n):
        out = f()
        k += int(not all(torch.equal(a, b) for a, b in zip(out, ref)))
    bad[name] = k


qkv = (torch.randn(t, 3 * heads * 128, device="cuda", generator=g) * 1.5).to(L.ELEM)
grid = ops.KVGrid(ext, win)
qg = ops.pad_tokens_to_grid(qkv, grid)
stress("natten", lambda: [ops.natten(qg, grid, heads, 128, 128, win)])
x0 = torch.randn(t, dim, device="cuda", generator=g)
lw, lb = torch.randn(dim, device="cuda", generator=g), torch.randn(dim, device="cuda", generator=g)
stress("layernorm", lambda: [ops.layernorm_bf16(x0, lw, lb)])
params = init_block_params(np.random.default_rng(0), dim, heads, "blk", zero_residual=False)
bw = prepare_block(params, "blk", heads)
ws = Workspace(ops.KVGrid(ext, win), bw)
rope = RopeTables(ext, dim // heads)


def blk():
    y = x0.clone()
    block_forward(y, bw, ws, rope, ext, win)
    return [y]


stress("block", blk, N // 2)
cfg = m.full_scale_config()
p = m.init_model_params(cfg, seed=0, zero_residual=False)
rng = np.random.default_rng(1)
st = m.WeatherState(0, torch.from_numpy(rng.standard_normal((cfg.surface_in, cfg.grid.rows, cfg.grid.cols)).astype(np.float32)).cuda(),
                    torch.from_numpy(rng.standard_normal((cfg.atmos_vars, cfg.levels, cfg.grid.rows, cfg.grid.cols)).astype(np.float32)).cuda())
stress("encode", lambda: [m.encode(st, p, cfg).tokens.device], 20)
lat = m.encode(st, p, cfg)
stress("decode", lambda: (lambda d: [d.surface.device, d.atmos.device])(m.decode(lat, p, cfg)), 20)
print("mismatches", bad)

# latitude bands (emulated ranks): separate copy and fused epilogue halo paths
from paper_2503_22235_b200.bands import rollout_banded
import paper_2503_22235_b200.rollout as R
cfg = m.mid_config()
pm = m.init_model_params(cfg, seed=7, zero_residual=False)
rng = np.random.default_rng(4)
stm = m.WeatherState(0, rng.standard_normal((cfg.surface_in, cfg.grid.rows, cfg.grid.cols)),
                     rng.standard_normal((cfg.atmos_vars, cfg.levels, cfg.grid.rows, cfg.grid.cols)))
latm = m.encode(stm, pm, cfg)
bad.clear()
stress("bands2", lambda: [rollout_banded(latm, (6, 1), pm, cfg, world=2).tokens.device], 30)
stress("bands2_fused", lambda: [rollout_banded(latm, (6, 1), pm, cfg, world=2, fused=True).tokens.device], 30)
stress("rollout_graph", lambda: [R.rollout(latm, (6, 6, 1), pm, cfg).tokens.device], 30)
print("mismatches", bad)
