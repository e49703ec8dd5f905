"""Parameter naming and seeded random initialisation, draw-for-draw identical to the reference.

init_block_params follows attention.py:105-139 and init_model_params model.py:190-273: the same PCG64
stream (`numpy.random.default_rng(seed)`), the same draw order and shapes, the same 1/sqrt(fan_in) scales
and the same zero_residual convention, so a given seed yields bit-identical float64 weights on both sides.
"""

from __future__ import annotations

import math

import numpy as np

from .config import DOWNSAMPLE_STAGES, MLP_EXPANSION, N_STATIC_FIELDS, PRIMARY_SOURCE, ModelConfig
from .errors import ConfigError
from .tensor import Tensor

BLOCK_PARAM_SUFFIXES = (
    "ln1.gain", "ln1.bias",
    "attn.wq", "attn.bq", "attn.wk", "attn.bk", "attn.wv", "attn.bv", "attn.wo", "attn.bo",
    "ln2.gain", "ln2.bias",
    "mlp.w1", "mlp.b1", "mlp.w2", "mlp.b2",
)


def block_param_names(prefix: str) -> list[str]:
    return [f"{prefix}.{s}" for s in BLOCK_PARAM_SUFFIXES]


def _param(a: np.ndarray) -> Tensor:
    return Tensor(a, requires_grad=True)


def init_block_params(rng: np.random.Generator, dim: int, heads: int, prefix: str,
                      zero_residual: bool = True) -> dict[str, Tensor]:
    if dim % heads:
        raise ConfigError(f"dim {dim} not divisible by heads {heads}")
    scale = 1.0 / math.sqrt(dim)
    width = MLP_EXPANSION * dim
    out_scale = 0.0 if zero_residual else scale
    w2_scale = 0.0 if zero_residual else 1.0 / math.sqrt(width)
    p: dict[str, Tensor] = {}
    # draw order matters: wq, wk, wv, wo, w1, w2
    p[f"{prefix}.ln1.gain"] = _param(np.ones(dim))
    p[f"{prefix}.ln1.bias"] = _param(np.zeros(dim))
    for name in ("wq", "wk", "wv"):
        p[f"{prefix}.attn.{name}"] = _param(rng.standard_normal((dim, dim)) * scale)
        p[f"{prefix}.attn.b{name[1]}"] = _param(np.zeros(dim))
    p[f"{prefix}.attn.wo"] = _param(rng.standard_normal((dim, dim)) * out_scale)
    p[f"{prefix}.attn.bo"] = _param(np.zeros(dim))
    p[f"{prefix}.ln2.gain"] = _param(np.ones(dim))
    p[f"{prefix}.ln2.bias"] = _param(np.zeros(dim))
    p[f"{prefix}.mlp.w1"] = _param(rng.standard_normal((dim, width)) * scale)
    p[f"{prefix}.mlp.b1"] = _param(np.zeros(width))
    p[f"{prefix}.mlp.w2"] = _param(rng.standard_normal((width, dim)) * w2_scale)
    p[f"{prefix}.mlp.b2"] = _param(np.zeros(dim))
    return {k: p[k] for k in block_param_names(prefix)}


def _conv(rng, shape, fan_in, p, name, scale=None):
    s = (1.0 / math.sqrt(fan_in)) if scale is None else scale
    p[name + ".w"] = _param(rng.standard_normal(shape) * s)
    p[name + ".b"] = _param(np.zeros(shape[1] if name.endswith(".up") else shape[0]))


def _res_pair(rng, prefix, ch, p):
    for j in range(2):
        for conv in ("conv1", "conv2"):
            _conv(rng, (ch, ch, 3, 3), ch * 9, p, f"{prefix}.res{j}.{conv}")


def _encoder(cfg: ModelConfig, rng, prefix: str, zero_residual: bool, p: dict) -> None:
    sfc_in = cfg.surface_in + N_STATIC_FIELDS
    atm_in = cfg.atmos_vars * cfg.level_patch
    _conv(rng, (cfg.stem_channels, sfc_in, 3, 3), sfc_in * 9, p, f"{prefix}.stem_sfc")
    _conv(rng, (cfg.stem_channels, atm_in, 3, 3), atm_in * 9, p, f"{prefix}.stem_atm")
    c_in = cfg.stem_channels
    for i, c_out in enumerate(cfg.stage_channels):
        _conv(rng, (c_out, c_in, 3, 3), c_in * 9, p, f"{prefix}.stage{i}.down")
        _res_pair(rng, f"{prefix}.stage{i}", c_out, p)
        c_in = c_out
    for i in range(cfg.enc_blocks):
        p.update(init_block_params(rng, cfg.hidden, cfg.heads, f"{prefix}.blk{i}", zero_residual))


def init_model_params(cfg: ModelConfig, seed: int = 0, zero_residual: bool = True,
                      extra_sources: tuple[str, ...] = ()) -> dict[str, Tensor]:
    rng = np.random.default_rng(seed)
    p: dict[str, Tensor] = {}
    _encoder(cfg, rng, "enc", zero_residual, p)
    for name in extra_sources:
        if name == PRIMARY_SOURCE:
            raise ConfigError("primary source already has the default encoder")
        _encoder(cfg, rng, f"enc_op.{name}", zero_residual, p)
    for hz in cfg.horizons:
        for i in range(cfg.proc_blocks):
            p.update(init_block_params(rng, cfg.hidden, cfg.heads, f"proc{hz}.blk{i}", zero_residual))
    for i in range(cfg.dec_blocks):
        p.update(init_block_params(rng, cfg.hidden, cfg.heads, f"dec.blk{i}", zero_residual))
    chans = [cfg.hidden, *cfg.stage_channels[-2::-1], cfg.stem_channels]
    for i in range(DOWNSAMPLE_STAGES):
        ci, co = chans[i], chans[i + 1]
        _conv(rng, (ci, co, 4, 4), ci * 16, p, f"dec.stage{i}.up")
        _res_pair(rng, f"dec.stage{i}", co, p)
    head = 0.0 if zero_residual else None
    _conv(rng, (cfg.surface_out, cfg.stem_channels, 3, 3), cfg.stem_channels * 9, p, "dec.head_sfc", head)
    atm_out = cfg.atmos_vars * cfg.level_patch
    _conv(rng, (atm_out, cfg.stem_channels, 3, 3), cfg.stem_channels * 9, p, "dec.head_atm", head)
    return p


def encoder_prefix(source: str) -> str:
    return "enc" if source == PRIMARY_SOURCE else f"enc_op.{source}"


def available_sources(params: dict) -> list[str]:
    names = [PRIMARY_SOURCE] if "enc.stem_sfc.w" in params else []
    for key in params:
        if key.startswith("enc_op."):
            src = key.split(".")[1]
            if src not in names:
                names.append(src)
    return names
