"""Model / grid configuration, field-for-field compatible with the reference.

Mirrors gridcast.grid.GridSpec (grid.py:25-53) and gridcast.model.ModelConfig (model.py:61-124) —
same fields, defaults, validation (ConfigError) and derived properties — plus the named configurations
(model.py:127-151), the key=value config file (model.py:527-607) and the dry-run shape plan
(model.py:456-520).  `mid_config` is the parity configuration of SURVEY.md §8d (depth bump, row bump and
column wrap at the paper's (5,7,7) window and dh = 128).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ConfigError

N_STATIC_FIELDS = 7
DOWNSAMPLE_STAGES = 3
PRIMARY_SOURCE = "primary"
MLP_EXPANSION = 4


@dataclass(frozen=True)
class GridSpec:
    rows: int
    cols: int
    north_lat: float = 90.0
    lat_step: float = 0.25
    lon_step: float = 0.25
    south_pole_omitted: bool = True
    planet_radius_km: float = 6371.0

    def __post_init__(self):
        checks = (
            (self.rows >= 1 and self.cols >= 1, f"grid extents must be positive, got {self.rows}x{self.cols}"),
            (self.lat_step > 0 and self.lon_step > 0, "grid steps must be positive"),
            (abs(self.cols * self.lon_step - 360.0) <= 1e-9,
             f"{self.cols} columns of {self.lon_step} deg do not close the circle"),
        )
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)
        southmost = self.north_lat - (self.rows - 1) * self.lat_step
        if self.north_lat > 90.0 + 1e-12 or southmost < -90.0 - 1e-12:
            raise ConfigError(f"grid rows span {southmost}..{self.north_lat}, beyond the poles")
        if self.south_pole_omitted and abs(southmost + 90.0) < 1e-12:
            raise ConfigError("south pole row present but declared omitted")
        if self.planet_radius_km <= 0:
            raise ConfigError("planet radius must be positive")

    @property
    def shape(self) -> tuple[int, int]:
        return (self.rows, self.cols)


def quarter_degree_grid() -> GridSpec:
    return GridSpec(rows=720, cols=1440, north_lat=90.0, lat_step=0.25, lon_step=0.25)


def desk_grid() -> GridSpec:
    return GridSpec(rows=40, cols=80, north_lat=90.0, lat_step=4.5, lon_step=4.5)


@dataclass(frozen=True)
class ModelConfig:
    grid: GridSpec
    surface_in: int = 4
    surface_out: int = 6
    atmos_vars: int = 3
    levels: int = 8
    level_patch: int = 4
    stem_channels: int = 16
    stage_channels: tuple = (24, 32, 48)
    hidden: int = 48
    heads: int = 4
    window: tuple = (3, 3, 3)
    enc_blocks: int = 2
    dec_blocks: int = 2
    proc_blocks: int = 4
    horizons: tuple = (1, 6)
    max_dt: int = 336

    def __post_init__(self):
        if self.levels % self.level_patch:
            raise ConfigError(f"levels {self.levels} not divisible by level patch {self.level_patch}")
        if len(self.stage_channels) != DOWNSAMPLE_STAGES:
            raise ConfigError(f"expected {DOWNSAMPLE_STAGES} stage channel counts")
        if self.stage_channels[-1] != self.hidden:
            raise ConfigError("last stage channels must equal the token width")
        if self.hidden % self.heads:
            raise ConfigError(f"hidden {self.hidden} not divisible by heads {self.heads}")
        dh = self.hidden // self.heads
        if dh % 2 or dh < 6:
            raise ConfigError(f"head dim {dh} must be even and at least 6 for rotary bands")
        factor = 1 << DOWNSAMPLE_STAGES
        if self.grid.rows % factor or self.grid.cols % factor:
            raise ConfigError(f"grid {self.grid.rows}x{self.grid.cols} not divisible by downsampling {factor}")
        ext = self.latent_extents
        if any(w > e for w, e in zip(self.window, ext)):
            raise ConfigError(f"attention window {self.window} exceeds latent extents {ext}")
        if min(self.surface_in, self.surface_out, self.atmos_vars) < 1:
            raise ConfigError("channel counts must be positive")
        if min(self.proc_blocks, self.enc_blocks, self.dec_blocks) < 1:
            raise ConfigError("block counts must be positive")
        if any(h < 1 for h in self.horizons) or len(set(self.horizons)) != len(self.horizons):
            raise ConfigError(f"invalid processor horizons {self.horizons}")
        if self.max_dt < 1:
            raise ConfigError("max_dt must be positive")

    @property
    def depth_planes(self) -> int:
        return 1 + self.levels // self.level_patch

    @property
    def latent_extents(self) -> tuple[int, int, int]:
        factor = 1 << DOWNSAMPLE_STAGES
        return (self.depth_planes, self.grid.rows // factor, self.grid.cols // factor)

    @property
    def tokens(self) -> int:
        return math.prod(self.latent_extents)

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


def desk_config() -> ModelConfig:
    return ModelConfig(grid=desk_grid())


def full_scale_config() -> ModelConfig:
    return ModelConfig(grid=quarter_degree_grid(), surface_in=8, surface_out=17, atmos_vars=5, levels=28,
                       level_patch=7, stem_channels=192, stage_channels=(256, 512, 1024), hidden=1024, heads=8,
                       window=(5, 7, 7), enc_blocks=2, dec_blocks=2, proc_blocks=10)


def tiny_config() -> ModelConfig:
    return ModelConfig(grid=GridSpec(rows=24, cols=24, lat_step=4.5, lon_step=15.0), surface_in=2,
                       surface_out=3, atmos_vars=2, levels=4, level_patch=2, stem_channels=6,
                       stage_channels=(6, 8, 12), hidden=12, heads=2, window=(3, 3, 3), enc_blocks=1,
                       dec_blocks=1, proc_blocks=2)


def mid_config() -> ModelConfig:
    """SURVEY.md §8d parity configuration: latent (7, 9, 18), dh 128, window (5, 7, 7)."""
    return ModelConfig(grid=GridSpec(72, 144, lat_step=2.5, lon_step=2.5), surface_in=8, surface_out=17,
                       atmos_vars=5, levels=12, level_patch=2, stem_channels=32, stage_channels=(64, 128, 256),
                       hidden=256, heads=2, window=(5, 7, 7), enc_blocks=2, dec_blocks=2, proc_blocks=10)


# ------------------------------------------------------------------------------------------------
# key = value config files (model.py:527-607)
# ------------------------------------------------------------------------------------------------
_GRID_KEYS = ("rows", "cols", "north_lat", "lat_step", "lon_step", "south_pole_omitted", "planet_radius_km")
_KEY_TYPES = {
    "rows": int, "cols": int, "north_lat": float, "lat_step": float, "lon_step": float,
    "south_pole_omitted": bool, "planet_radius_km": float, "surface_in": int, "surface_out": int,
    "atmos_vars": int, "levels": int, "level_patch": int, "stem_channels": int, "stage_channels": tuple,
    "hidden": int, "heads": int, "window": tuple, "enc_blocks": int, "dec_blocks": int, "proc_blocks": int,
    "horizons": tuple, "max_dt": int,
}


def config_to_dict(cfg: ModelConfig) -> dict:
    out = {k: getattr(cfg.grid, k) for k in _GRID_KEYS}
    for k in _KEY_TYPES:
        if k not in _GRID_KEYS:
            out[k] = getattr(cfg, k)
    return out


def config_from_dict(d: dict) -> ModelConfig:
    grid = GridSpec(**{k: d[k] for k in _GRID_KEYS})
    rest = {k: v for k, v in d.items() if k in _KEY_TYPES and k not in _GRID_KEYS}
    return ModelConfig(grid=grid, **rest)


_FOREIGN: dict = {}


def as_config(cfg) -> ModelConfig:
    """Our ModelConfig for `cfg`: itself, or the field-for-field equal copy of another package's config (the
    reference's gridcast.model.ModelConfig has the same fields but not every derived property used here, e.g.
    head_dim), built once per distinct config.  Validation as ModelConfig (ConfigError)."""
    if isinstance(cfg, ModelConfig):
        return cfg
    hit = _FOREIGN.get(cfg)
    if hit is None:
        d = {k: getattr(cfg.grid, k) for k in _GRID_KEYS}
        d.update({k: getattr(cfg, k) for k in _KEY_TYPES if k not in _GRID_KEYS})
        hit = _FOREIGN[cfg] = config_from_dict(d)
    return hit


def _fmt(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, tuple):
        return ",".join(str(e) for e in v)
    return str(v)


def save_config(path, cfg: ModelConfig) -> None:
    with open(path, "w") as f:
        for k, v in config_to_dict(cfg).items():
            f.write(f"{k} = {_fmt(v)}\n")


def _parse(ty, raw: str):
    if ty is bool:
        if raw not in ("true", "false"):
            raise ValueError(raw)
        return raw == "true"
    if ty is tuple:
        return tuple(int(e) for e in raw.split(","))
    return ty(raw)


def load_config(path) -> ModelConfig:
    vals: dict = {}
    with open(path) as f:
        for lineno, raw in enumerate(f, 1):
            text = raw.split("#", 1)[0].strip()
            if not text:
                continue
            key, sep, val = text.partition("=")
            if not sep:
                raise ConfigError(f"{path}:{lineno}: expected key = value")
            key, val = key.strip(), val.strip()
            if key not in _KEY_TYPES:
                raise ConfigError(f"{path}:{lineno}: unknown key {key!r}")
            try:
                vals[key] = _parse(_KEY_TYPES[key], val)
            except ValueError:
                raise ConfigError(f"{path}:{lineno}: bad value {val!r} for {key}") from None
    missing = sorted(set(_KEY_TYPES) - set(vals))
    if missing:
        raise ConfigError(f"{path}: missing keys {missing}")
    return config_from_dict(vals)


# ------------------------------------------------------------------------------------------------
# dry-run shape arithmetic (model.py:456-520)
# ------------------------------------------------------------------------------------------------
def _conv_n(co, ci, k):
    return co * ci * k * k + co


def _block_n(dim):
    return 4 * dim + 4 * (dim * dim + dim) + dim * MLP_EXPANSION * dim + MLP_EXPANSION * dim \
        + MLP_EXPANSION * dim * dim + dim


def shape_plan(cfg: ModelConfig) -> dict:
    g = cfg.grid
    stages, r, c = [], g.rows, g.cols
    for i, ch in enumerate(cfg.stage_channels):
        r, c = r // 2, c // 2
        stages.append({"stage": i, "channels": ch, "rows": r, "cols": c})
    n = _conv_n(cfg.stem_channels, cfg.surface_in + N_STATIC_FIELDS, 3) \
        + _conv_n(cfg.stem_channels, cfg.atmos_vars * cfg.level_patch, 3)
    ci = cfg.stem_channels
    for ch in cfg.stage_channels:
        n += _conv_n(ch, ci, 3) + 4 * _conv_n(ch, ch, 3)
        ci = ch
    n += (cfg.enc_blocks + cfg.dec_blocks + len(cfg.horizons) * cfg.proc_blocks) * _block_n(cfg.hidden)
    chans = [cfg.hidden] + list(cfg.stage_channels[-2::-1]) + [cfg.stem_channels]
    for i in range(DOWNSAMPLE_STAGES):
        n += chans[i] * chans[i + 1] * 16 + chans[i + 1] + 4 * _conv_n(chans[i + 1], chans[i + 1], 3)
    n += _conv_n(cfg.surface_out, cfg.stem_channels, 3) + _conv_n(cfg.atmos_vars * cfg.level_patch,
                                                                  cfg.stem_channels, 3)
    wd, wh, ww = cfg.window
    return {
        "grid": (g.rows, g.cols),
        "surface_input": (cfg.surface_in + N_STATIC_FIELDS, g.rows, g.cols),
        "atmos_input": (cfg.atmos_vars, cfg.levels, g.rows, g.cols),
        "level_groups": cfg.levels // cfg.level_patch,
        "plane_channels_in": cfg.atmos_vars * cfg.level_patch,
        "stages": stages,
        "latent_extents": cfg.latent_extents,
        "tokens": cfg.tokens,
        "token_width": cfg.hidden,
        "window": cfg.window,
        "attention_keys": wd * wh * ww,
        "blocks_total": cfg.enc_blocks + cfg.dec_blocks + len(cfg.horizons) * cfg.proc_blocks,
        "surface_output": (cfg.surface_out, g.rows, g.cols),
        "atmos_output": (cfg.atmos_vars, cfg.levels, g.rows, g.cols),
        "param_elements": n,
    }


def conv_flops(cfg: ModelConfig) -> dict:
    """Algorithmic FLOPs (2 x multiply-adds) of the encoder and decoder pyramids of one forecast, all depth planes
    (model.py:296-325, 363-421): 3x3 convs 2 * P_out * Cout * 9 * Cin; the stride-2 transposed 4x4 conv
    2 * P_out * Cout * 4 * Cin (each output pixel sees 2 x 2 taps); heads 192 -> surface_out (plane 0) and
    -> atmos_vars * level_patch (level-group planes)."""
    g = cfg.grid
    groups = cfg.levels // cfg.level_patch
    planes = 1 + groups
    enc = 2.0 * g.rows * g.cols * cfg.stem_channels * 9 * ((cfg.surface_in + N_STATIC_FIELDS)
                                                           + groups * cfg.atmos_vars * cfg.level_patch)
    r, c, ci = g.rows, g.cols, cfg.stem_channels
    for ch in cfg.stage_channels:
        r, c = r // 2, c // 2
        enc += planes * 2.0 * r * c * ch * 9 * (ci + 4 * ch)  # stride-2 down + two res blocks (2 convs each)
        ci = ch
    dec = 0.0
    chans = [cfg.hidden] + list(cfg.stage_channels[-2::-1]) + [cfg.stem_channels]
    for i in range(DOWNSAMPLE_STAGES):
        r, c = r * 2, c * 2
        dec += planes * 2.0 * r * c * chans[i + 1] * (4 * chans[i] + 4 * 9 * chans[i + 1])
    dec += 2.0 * g.rows * g.cols * 9 * cfg.stem_channels * (cfg.surface_out + groups * cfg.atmos_vars * cfg.level_patch)
    return {"encode_conv": enc, "decode_conv": dec}
