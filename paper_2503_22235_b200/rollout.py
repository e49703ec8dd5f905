"""Greedy mixed-horizon latent rollout (gridcast/rollout.py), drop-in on the B200 path.

The plan is validated in full before any launch (rollout.py:48-53).  The latent is copied once into a
device buffer and every processor step runs in place on it; no encode/decode happens inside the rollout.
With `graphs=True` (default for plans of more than one step) each distinct horizon's step is captured once
as a CUDA graph and replayed, so a 14-day forecast issues 56 graph launches instead of ~4.5k kernels.
`engine` (the reference's activation-offload engine for training) is accepted and ignored: the inference
forward keeps no activations to offload, so results are identical with or without it.
"""

from __future__ import annotations

import torch

from .errors import ConfigError
from .model import (CALL_COUNTS, PRIMARY_SOURCE, DecodedFields, LatentState, ModelConfig, WeatherState,
                    _check_processor, _tokens, decode, encode, process_inplace)
from .tensor import Tensor

__all__ = ["greedy_plan", "plan_hours", "rollout", "forecast"]


def greedy_plan(dt: int, max_dt: int = 336) -> tuple:
    """Sixes first, then ones (rollout.py:33-41)."""
    if isinstance(dt, bool) or not isinstance(dt, int):
        raise ConfigError(f"dt must be an integer hour count, got {dt!r}")
    if dt < 0:
        raise ConfigError(f"dt must be nonnegative, got {dt}")
    if dt > max_dt:
        raise ConfigError(f"dt {dt} exceeds the configured cap {max_dt}")
    sixes, ones = divmod(dt, 6)
    return (6,) * sixes + (1,) * ones


def plan_hours(plan) -> int:
    return sum(plan)


class _Rollout:
    """Per (params, cfg): one resident token buffer and a CUDA graph per horizon captured on it."""

    def __init__(self, params: dict, cfg: ModelConfig):
        self.params, self.cfg = params, cfg
        self.buf = torch.zeros((cfg.tokens, cfg.hidden), dtype=torch.float32, device="cuda")
        self.graphs: dict = {}

    def graph(self, horizon: int) -> torch.cuda.CUDAGraph:
        g = self.graphs.get(horizon)
        if g is None:
            # warm-up outside capture: weight conversion, workspaces, kernel attributes
            process_inplace(self.buf, self.params, self.cfg, horizon)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                process_inplace(self.buf, self.params, self.cfg, horizon)
            # the graph holds raw device pointers: keep the captured weights alive with it
            from .runtime import CACHE
            self.keep = getattr(self, "keep", []) + [CACHE.block(self.params, f"proc{horizon}.blk{i}", self.cfg.heads)
                                                    for i in range(self.cfg.proc_blocks)]
            self.graphs[horizon] = g
        return g


_ROLLOUTS: dict = {}


def _rollout_state(params: dict, cfg: ModelConfig) -> _Rollout:
    from .model import device_model
    fp = device_model(params, cfg)._fp  # parameter arrays' identities: new arrays -> new graphs
    key = (id(params), cfg)
    r = _ROLLOUTS.get(key)
    if r is None or r.params is not params or getattr(r, "fp", None) != fp:
        r = _Rollout(params, cfg)
        r.fp = fp
        _ROLLOUTS[key] = r
    return r


def rollout(lat: LatentState, plan, params: dict, cfg: ModelConfig, engine=None,
            graphs: bool | None = None) -> LatentState:
    """Apply the plan's processors in sequence, entirely in latent space (rollout.py:56-81)."""
    plan = tuple(plan)
    for h in plan:
        if h not in cfg.horizons:
            raise ConfigError(f"plan step {h} h not among configured horizons {cfg.horizons}")
        _check_processor(params, cfg, h)
    if not plan:
        return lat
    use_graphs = (len(plan) > 1) if graphs is None else graphs
    if use_graphs:
        from .model import device_model
        device_model(params, cfg)  # refresh converted weights if the caller changed parameters
        st = _rollout_state(params, cfg)
        steps = {h: st.graph(h) for h in sorted(set(plan))}
        st.buf.copy_(_tokens(lat))
        for h in plan:
            steps[h].replay()
            CALL_COUNTS[f"process{h}"] += 1
        x = st.buf.clone()
    else:
        x = _tokens(lat).clone()
        for h in plan:
            CALL_COUNTS[f"process{h}"] += 1
            process_inplace(x, params, cfg, h)
    return LatentState(Tensor(device=x), lat.valid_time + plan_hours(plan), tuple(lat.extents))


def forecast(state: WeatherState, dt: int, params: dict, cfg: ModelConfig, source: str = PRIMARY_SOURCE,
             engine=None) -> DecodedFields:
    """encode -> greedy latent rollout -> decode (rollout.py:84-91)."""
    plan = greedy_plan(dt, cfg.max_dt)
    lat = encode(state, params, cfg, source=source)
    lat = rollout(lat, plan, params, cfg, engine=engine)
    return decode(lat, params, cfg)
