"""Greedy mixed-horizon latent rollout (gridcast/rollout.py), drop-in on the B200 path.

The plan is validated in full before any launch (rollout.py:48-53).  The latent is copied once into a
device buffer and every processor step runs in place on it; no encode/decode happens inside the rollout.
With `graphs=True` (default for plans of more than one step) each distinct horizon's step is captured once
as a CUDA graph and replayed, so a 14-day forecast issues 56 graph launches instead of ~4.5k kernels.
`engine` (the reference's activation-offload engine for training) is accepted and ignored: the inference
forward keeps no activations to offload, so results are identical with or without it.

Ensembles ("8-member ensemble batch"): `rollout_ensemble` / `forecast_ensemble`
stack the members' latents member-major in one (members * T, hidden) buffer and run every processor block
once for all of them (GEMMs over members * T rows, attention with a member index so windows never cross
members).  Each member's result is bitwise the single-member rollout of the same latent.
"""

from __future__ import annotations

import torch

from .config import as_config
from .errors import ConfigError
from .model import (CALL_COUNTS, PRIMARY_SOURCE, DecodedFields, LatentState, ModelConfig, WeatherState,
                    _check_processor, check_latent, decode, encode, latent_tokens, process_inplace)
from .tensor import Tensor

__all__ = ["greedy_plan", "plan_hours", "rollout", "forecast", "rollout_ensemble", "forecast_ensemble",
           "perturbed_members"]


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
    """Per (params, cfg, members): one resident token buffer and a CUDA graph per horizon captured on it."""

    def __init__(self, params: dict, cfg: ModelConfig, members: int = 1):
        self.params, self.cfg, self.members = params, cfg, int(members)
        self.buf = torch.zeros((self.members * cfg.tokens, cfg.hidden), dtype=torch.float32, device="cuda")
        self.graphs: dict = {}

    def graph(self, horizon: int) -> torch.cuda.CUDAGraph:
        g = self.graphs.get(horizon)
        if g is None:
            # warm-up outside capture: weight conversion, workspaces, kernel attributes
            process_inplace(self.buf, self.params, self.cfg, horizon, self.members)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                process_inplace(self.buf, self.params, self.cfg, horizon, self.members)
            # the graph holds raw device pointers: keep the captured weights alive with it
            from .runtime import CACHE
            self.keep = getattr(self, "keep", []) + [CACHE.block(self.params, f"proc{horizon}.blk{i}", self.cfg.heads)
                                                    for i in range(self.cfg.proc_blocks)]
            self.graphs[horizon] = g
        return g


_ROLLOUTS: dict = {}


def _rollout_state(params: dict, cfg: ModelConfig, members: int = 1) -> _Rollout:
    from .model import device_model
    fp = device_model(params, cfg)._fp  # parameter arrays' identities: new arrays -> new graphs
    key = (id(params), cfg, int(members))
    r = _ROLLOUTS.get(key)
    if r is None or r.params is not params or getattr(r, "fp", None) != fp:
        r = _Rollout(params, cfg, members)
        r.fp = fp
        _ROLLOUTS[key] = r
    return r


def _check_plan(plan, params: dict, cfg: ModelConfig) -> tuple:
    plan = tuple(plan)
    for h in plan:
        if h not in cfg.horizons:
            raise ConfigError(f"plan step {h} h not among configured horizons {cfg.horizons}")
        _check_processor(params, cfg, h)
    return plan


def rollout(lat: LatentState, plan, params: dict, cfg: ModelConfig, engine=None,
            graphs: bool | None = None) -> LatentState:
    """Apply the plan's processors in sequence, entirely in latent space (rollout.py:56-81)."""
    cfg = as_config(cfg)
    plan = _check_plan(plan, params, cfg)
    if not plan:
        return lat
    x0 = latent_tokens(lat, cfg)
    use_graphs = (len(plan) > 1) if graphs is None else graphs
    if use_graphs:
        from .model import device_model
        device_model(params, cfg)  # refresh converted weights if the caller changed parameters
        st = _rollout_state(params, cfg)
        steps = {h: st.graph(h) for h in sorted(set(plan))}
        st.buf.copy_(x0)
        for h in plan:
            steps[h].replay()
            CALL_COUNTS[f"process{h}"] += 1
        x = st.buf.clone()
    else:
        x = x0.clone()
        for h in plan:
            CALL_COUNTS[f"process{h}"] += 1
            process_inplace(x, params, cfg, h)
    return LatentState(Tensor(device=x), lat.valid_time + plan_hours(plan), tuple(lat.extents))


def forecast(state: WeatherState, dt: int, params: dict, cfg: ModelConfig, source: str = PRIMARY_SOURCE,
             engine=None, host_out=None) -> DecodedFields:
    """encode -> greedy latent rollout -> decode (rollout.py:84-91).  host_out: see model.decode (the fields
    stream to page-locked host tensors while the decoder runs)."""
    cfg = as_config(cfg)
    plan = greedy_plan(dt, cfg.max_dt)
    lat = encode(state, params, cfg, source=source)
    lat = rollout(lat, plan, params, cfg, engine=engine)
    return decode(lat, params, cfg, host_out=host_out)


def rollout_ensemble(latents, plan, params: dict, cfg: ModelConfig, graphs: bool = True) -> list:
    """rollout() of every member at once: one (members * T, hidden) batch through each processor block.

    Validation as rollout() (before any launch); an empty plan returns the input objects.  Member m's output
    equals rollout(latents[m], plan, ...) bitwise."""
    cfg = as_config(cfg)
    latents = list(latents)
    plan = _check_plan(plan, params, cfg)
    if not latents:
        raise ConfigError("ensemble of zero members")
    for lt in latents:
        check_latent(lt, cfg)
    if not plan:
        return latents
    from .model import device_model
    device_model(params, cfg)
    n, t = len(latents), cfg.tokens
    st = _rollout_state(params, cfg, n)
    steps = {h: st.graph(h) for h in sorted(set(plan))} if graphs else {}  # capture warm-up runs on st.buf
    for m, lt in enumerate(latents):
        st.buf[m * t:(m + 1) * t].copy_(latent_tokens(lt, cfg))
    if graphs:
        for h in plan:
            steps[h].replay()
            CALL_COUNTS[f"process{h}"] += n
    else:
        for h in plan:
            process_inplace(st.buf, params, cfg, h, n)
            CALL_COUNTS[f"process{h}"] += n
    hours = plan_hours(plan)
    return [LatentState(Tensor(device=st.buf[m * t:(m + 1) * t].clone()), lt.valid_time + hours, tuple(lt.extents))
            for m, lt in enumerate(latents)]


def forecast_ensemble(states, dt: int, params: dict, cfg: ModelConfig, source: str = PRIMARY_SOURCE,
                      host_outs=None) -> list:
    """forecast() of every member: per-member encode, one batched greedy rollout, per-member decode.
    host_outs: per-member (surface, atmos) page-locked host buffers the decoded fields stream to (model.decode)."""
    cfg = as_config(cfg)
    plan = greedy_plan(dt, cfg.max_dt)
    lats = [encode(s, params, cfg, source=source) for s in states]
    lats = rollout_ensemble(lats, plan, params, cfg)
    if host_outs is None:
        host_outs = [None] * len(lats)
    return [decode(lt, params, cfg, host_out=h) for lt, h in zip(lats, host_outs)]


def perturbed_members(state: WeatherState, members: int, scale: float = 0.01, seed: int = 100) -> list:
    """Ensemble initial states: member m = state + N(0, scale) from default_rng(seed + m), in the style of
    the reference's perturbed sources (synthdata.py:186-193)."""
    import numpy as np
    from .tensor import host_array
    sfc, atm = host_array(state.surface), host_array(state.atmos)
    out = []
    for m in range(members):
        rng = np.random.default_rng(seed + m)
        ds = rng.standard_normal(sfc.shape, dtype=np.float32 if sfc.dtype == np.float32 else np.float64)
        da = rng.standard_normal(atm.shape, dtype=np.float32 if atm.dtype == np.float32 else np.float64)
        out.append(WeatherState(state.valid_time, sfc + scale * ds, atm + scale * da))
    return out
