"""Drop-in model API (gridcast/model.py): encode / process / decode on the B200 path.

Same signatures, state types, error behaviour (ConfigError before any launch) and CALL_COUNTS
instrumentation as the reference (model.py:53-58, 158-183, 363-449).  The latent lives on the device as an
fp32 (T, hidden) token grid; decoded fields are fp32 device tensors exposed through `.values` (float64
numpy on first access) so reference callers keep working.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from .blocks import block_forward
from .config import (DOWNSAMPLE_STAGES, as_config, N_STATIC_FIELDS, PRIMARY_SOURCE, GridSpec, ModelConfig,  # noqa: F401
                     config_from_dict, config_to_dict, desk_config, full_scale_config, load_config, mid_config,
                     save_config, shape_plan, tiny_config)
from .errors import ConfigError
from .grid import desk_grid, quarter_degree_grid, static_fields  # noqa: F401
from .params import (available_sources, block_param_names, encoder_prefix, init_block_params,  # noqa: F401
                     init_model_params)
from .pyramid import (DecoderWeights, EncoderWeights, PyramidBuffers, check_input_range, decode_planes,
                      encode_planes)
from .runtime import CACHE
from .tensor import Tensor, content_tag, host_array, host_values

__all__ = [
    "ModelConfig", "desk_config", "full_scale_config", "tiny_config", "mid_config", "WeatherState",
    "DecodedFields", "LatentState", "init_model_params", "encode", "process", "decode", "blend_latents",
    "encoder_prefix", "available_sources", "shape_plan", "save_config", "load_config", "CALL_COUNTS",
    "reset_call_counts", "device_model",
]

CALL_COUNTS = {"encode": 0, "process1": 0, "process6": 0, "decode": 0}


def reset_call_counts() -> None:
    for k in CALL_COUNTS:
        CALL_COUNTS[k] = 0


@dataclass
class WeatherState:
    """Gridded fields at one valid time (model.py:158-163): surface (C, H, W), atmos (A, L, H, W)."""
    valid_time: int
    surface: object
    atmos: object


@dataclass
class DecodedFields:
    """Decoder output (model.py:166-175); surface / atmos are device-backed Tensors."""
    valid_time: int
    surface: Tensor
    atmos: Tensor

    def to_state(self) -> WeatherState:
        return WeatherState(self.valid_time, self.surface.values.copy(), self.atmos.values.copy())

    def to_host(self, out=None):
        """(surface, atmos) as float32 host tensors in page-locked memory (one DMA each, no float64 widening).
        Pass `out` = a previous result to reuse its pinned buffers (steady-state: no host allocation).  Fields
        decoded with decode(..., host_out=out) are already streamed there: this only waits for the copies."""
        if out is not None and getattr(self, "_host", None) is out:
            torch.cuda.current_stream().synchronize()
            return out
        if out is None:
            out = tuple(torch.empty(t.device.shape, dtype=torch.float32, pin_memory=True)
                        for t in (self.surface, self.atmos))
        for host, t in zip(out, (self.surface, self.atmos)):
            host.copy_(t.device, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out


@dataclass
class LatentState:
    """Token grid between encoder and decoder (model.py:178-183); tokens (T, hidden) fp32 on the device."""
    tokens: Tensor
    valid_time: int
    extents: tuple


# ------------------------------------------------------------------------------------------------
# device-resident model
# ------------------------------------------------------------------------------------------------
class DeviceModel:
    """Everything the forward needs on the device for one (params, cfg): converted weights (lazily, per
    encoder source / block / decoder), activation buffers and rotary tables."""

    def __init__(self, params: dict, cfg: ModelConfig):
        self.params = params
        self.cfg = cfg
        self._enc: dict = {}
        self._dec = None
        self._bufs = None

    def fingerprint(self, prefix: str | None = None, blocks: bool = True) -> tuple:
        """Content tags (tensor.content_tag) of the parameters named `prefix.*` (all with None; without the
        `.blk*` transformer blocks when blocks=False — runtime.CACHE checks those per block).  Scoped so a call
        checks only the arrays it uses: tagging all ~450 arrays of the full model costs ~5-10 ms of host time,
        which left the GPU idle at the start of every encode / process / decode."""
        return tuple(content_tag(v) for k, v in self.params.items()
                     if (prefix is None or k.startswith(prefix + ".")) and (blocks or ".blk" not in k))

    def refresh(self) -> None:
        """Drop the converted pyramid weights whose host arrays changed (kept for callers that want an explicit
        check; encoder() / decoder() check their own arrays on every access)."""
        for pre in list(self._enc):
            if self._enc[pre][0] != self.fingerprint(pre, blocks=False):
                del self._enc[pre]
        if self._dec is not None and self._dec[0] != self.fingerprint("dec", blocks=False):
            self._dec = None

    @property
    def _fp(self) -> tuple:
        """Content tags of the processor blocks (what the captured rollout graphs hold)."""
        return tuple(content_tag(v) for k, v in self.params.items() if k.startswith("proc"))

    def encoder(self, prefix: str) -> EncoderWeights:
        fp = self.fingerprint(prefix, blocks=False)
        hit = self._enc.get(prefix)
        if hit is None or hit[0] != fp:
            hit = self._enc[prefix] = (fp, EncoderWeights(self.params, prefix))
        return hit[1]

    def decoder(self) -> DecoderWeights:
        fp = self.fingerprint("dec", blocks=False)
        if self._dec is None or self._dec[0] != fp:
            self._dec = (fp, DecoderWeights(self.params))
        return self._dec[1]

    def buffers(self) -> PyramidBuffers:
        if self._bufs is None:
            self._bufs = PyramidBuffers(self.cfg)
        return self._bufs

    def run_blocks(self, x: torch.Tensor, prefixes, batch: int = 1) -> None:
        """Blocks in place on x: (batch * tokens, hidden), `batch` independent latents stacked member-major."""
        cfg = self.cfg
        ext = cfg.latent_extents
        rope = CACHE.rope(ext, cfg.head_dim)
        for i, pre in enumerate(prefixes):
            bw = CACHE.block(self.params, pre, cfg.heads)
            # folded LayerNorm: block i > 0 finds x's fp16 copy and row statistics left by block i-1's W2
            block_forward(x, bw, CACHE.workspace(ext, cfg.window, bw, batch=batch), rope, ext, cfg.window,
                          prepped=i > 0)


_models: dict = {}
_mlock = threading.Lock()


def device_model(params: dict, cfg: ModelConfig) -> DeviceModel:
    key = (id(params), cfg)
    with _mlock:
        hit = _models.get(key)
        if hit is None or hit.params is not params:
            hit = DeviceModel(params, cfg)
            _models[key] = hit
    return hit


def _to_device(a, shape) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to("cuda", torch.float32)
    return torch.from_numpy(np.ascontiguousarray(host_array(a, np.float32))).to("cuda")


def _tokens(lat: LatentState) -> torch.Tensor:
    t = lat.tokens
    if isinstance(t, Tensor) and t.device is not None:
        return t.device
    if isinstance(t, torch.Tensor):
        return t.to("cuda", torch.float32)
    return torch.from_numpy(np.ascontiguousarray(host_values(t), dtype=np.float32)).to("cuda")


def check_latent(lat: LatentState, cfg: ModelConfig) -> None:
    """The latent must be the configuration's token grid: the kernels take their sizes from cfg, so a
    mismatched latent would read / write out of bounds.  ConfigError before any launch, as the reference's
    natten_block check (attention.py:150-151) would raise inside its first block."""
    ext = tuple(int(e) for e in lat.extents)
    if ext != tuple(cfg.latent_extents):
        raise ConfigError(f"latent extents {ext} != config latent extents {tuple(cfg.latent_extents)}")
    shape = tuple(lat.tokens.shape)
    if shape != (cfg.tokens, cfg.hidden):
        raise ConfigError(f"latent tokens {shape} != (prod of extents {ext}, hidden) = {(cfg.tokens, cfg.hidden)}")


def latent_tokens(lat: LatentState, cfg: ModelConfig) -> torch.Tensor:
    """Validated (check_latent) contiguous fp32 device tokens of a latent (no copy when already so)."""
    check_latent(lat, cfg)
    return _tokens(lat).to(torch.float32).contiguous()


def check_token_buffer(x: torch.Tensor, cfg: ModelConfig, batch: int = 1) -> None:
    """A device token buffer the blocks run in place on: (batch * tokens, hidden) contiguous fp32 CUDA."""
    want = (int(batch) * cfg.tokens, cfg.hidden)
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise ConfigError("token buffer must be a contiguous float32 CUDA tensor")
    if tuple(x.shape) != want:
        raise ConfigError(f"token buffer {tuple(x.shape)} != {want}")


# ------------------------------------------------------------------------------------------------
# API
# ------------------------------------------------------------------------------------------------
def stage_inputs(state: WeatherState, params: dict, cfg: ModelConfig, source: str = PRIMARY_SOURCE,
                 upload: bool = True):
    """encode()'s validation (ConfigError before any launch) and the host->device copy of the state into the
    pyramid input buffers; returns (device model, encoder weight prefix)."""
    cfg = as_config(cfg)
    prefix = encoder_prefix(source)
    if f"{prefix}.stem_sfc.w" not in params:
        raise ConfigError(f"no encoder for source {source!r}")
    g = cfg.grid
    if tuple(state.surface.shape) != (cfg.surface_in, g.rows, g.cols):
        raise ConfigError(f"surface shape {tuple(state.surface.shape)} != {(cfg.surface_in, g.rows, g.cols)}")
    if tuple(state.atmos.shape) != (cfg.atmos_vars, cfg.levels, g.rows, g.cols):
        raise ConfigError(f"atmos shape {tuple(state.atmos.shape)} != "
                          f"{(cfg.atmos_vars, cfg.levels, g.rows, g.cols)}")
    CALL_COUNTS["encode"] += 1
    dm = device_model(params, cfg)
    bufs = dm.buffers()
    if not bufs.statics_ready:
        bufs.sfc_in[cfg.surface_in:] = torch.from_numpy(static_fields(g).astype(np.float32)).to("cuda")
        bufs.statics_ready = True
    if not upload:
        return dm, prefix  # encode() streams the planes in (_stream_inputs)
    bufs.sfc_in[:cfg.surface_in].copy_(_to_device(state.surface, None), non_blocking=True)
    bufs.atm_in.copy_(_to_device(state.atmos, None), non_blocking=True)
    return dm, prefix


def _pinned_f32(a) -> bool:
    return isinstance(a, torch.Tensor) and a.device.type == "cpu" and a.dtype == torch.float32 and a.is_pinned() \
        and a.is_contiguous()


def _stream_inputs(state: WeatherState, bufs, cfg: ModelConfig) -> list:
    """Page-locked host fields -> the pyramid input buffers on the copy stream, one event per depth plane (surface,
    then each atmosphere level group: one contiguous run of levels per variable)."""
    main, side = torch.cuda.current_stream(), _copy_stream()
    side.wait_stream(main)  # the input buffers are free once earlier work on them is done
    p = cfg.level_patch
    evs = []
    with torch.cuda.stream(side):
        bufs.sfc_in[:cfg.surface_in].copy_(state.surface, non_blocking=True)
        evs.append(torch.cuda.Event())
        evs[-1].record(side)
        for g_ in range(cfg.levels // p):
            for a in range(cfg.atmos_vars):
                bufs.atm_in[a, g_ * p:(g_ + 1) * p].copy_(state.atmos[a, g_ * p:(g_ + 1) * p], non_blocking=True)
            evs.append(torch.cuda.Event())
            evs[-1].record(side)
    return evs


def encode(state: WeatherState, params: dict, cfg: ModelConfig, source: str = PRIMARY_SOURCE) -> LatentState:
    """Lift one gridded state into the latent token grid (model.py:363-390)."""
    cfg = as_config(cfg)
    streamed = _pinned_f32(state.surface) and _pinned_f32(state.atmos)
    dm, prefix = stage_inputs(state, params, cfg, source, upload=not streamed)
    bufs = dm.buffers()
    tokens = torch.empty((cfg.tokens, cfg.hidden), dtype=torch.float32, device="cuda")
    if streamed:
        # page-locked fields: plane q + 1 uploads on the copy stream while plane q's stem convolution runs
        evs = _stream_inputs(state, bufs, cfg)
        main = torch.cuda.current_stream()
        encode_planes(dm.encoder(prefix), bufs, cfg, tokens, before_plane=lambda q: main.wait_event(evs[q]))
        evs[-1].synchronize()  # the caller may reuse its host buffers once encode() returns
    else:
        encode_planes(dm.encoder(prefix), bufs, cfg, tokens)
    check_input_range(bufs)
    dm.run_blocks(tokens, [f"{prefix}.blk{i}" for i in range(cfg.enc_blocks)])
    return LatentState(Tensor(device=tokens), state.valid_time, cfg.latent_extents)


def _check_processor(params: dict, cfg: ModelConfig, horizon: int) -> None:
    if horizon not in cfg.horizons:
        raise ConfigError(f"no {horizon} h processor in config horizons {cfg.horizons}")
    if f"proc{horizon}.blk0.ln1.gain" not in params:
        raise ConfigError(f"parameters carry no {horizon} h processor")


def process_inplace(x: torch.Tensor, params: dict, cfg: ModelConfig, horizon: int, batch: int = 1) -> None:
    """proc_blocks blocks applied in place to a device token buffer (no validation, no counters); x holds
    `batch` latents stacked member-major ((batch * tokens, hidden))."""
    cfg = as_config(cfg)
    check_token_buffer(x, cfg, batch)
    device_model(params, cfg).run_blocks(x, [f"proc{horizon}.blk{i}" for i in range(cfg.proc_blocks)], batch)


def process(lat: LatentState, params: dict, cfg: ModelConfig, horizon: int) -> LatentState:
    """Advance the latent state by one processor application (model.py:393-405)."""
    cfg = as_config(cfg)
    _check_processor(params, cfg, horizon)
    x = latent_tokens(lat, cfg).clone()
    CALL_COUNTS[f"process{horizon}"] += 1
    process_inplace(x, params, cfg, horizon)
    return LatentState(Tensor(device=x), lat.valid_time + horizon, lat.extents)


_copy_streams: dict = {}


def _copy_stream() -> torch.cuda.Stream:
    dev = torch.cuda.current_device()
    if dev not in _copy_streams:
        _copy_streams[dev] = torch.cuda.Stream()
    return _copy_streams[dev]


def decode(lat: LatentState, params: dict, cfg: ModelConfig, host_out=None) -> DecodedFields:
    """Project the latent token grid back to gridded fields (model.py:408-421).

    host_out = (surface, atmos) page-locked float32 host tensors of the fields' shapes (e.g. a previous
    DecodedFields.to_host() result): the full-resolution decoder stage then runs plane by plane and each plane's
    fields are copied out on a side stream while the next plane is convolved (the device->host transfer hides
    behind the decoder); the returned fields' to_host(host_out) only waits."""
    cfg = as_config(cfg)
    x = latent_tokens(lat, cfg).clone()
    CALL_COUNTS["decode"] += 1
    dm = device_model(params, cfg)
    g = cfg.grid
    sshape, ashape = (cfg.surface_out, g.rows, g.cols), (cfg.atmos_vars, cfg.levels, g.rows, g.cols)
    if host_out is not None:
        hs, ha = host_out
        if tuple(hs.shape) != sshape or tuple(ha.shape) != ashape or hs.dtype != torch.float32 or \
                ha.dtype != torch.float32 or hs.device.type != "cpu" or ha.device.type != "cpu":
            raise ConfigError(f"host_out must be float32 host tensors of shapes {sshape} and {ashape}")
    dm.run_blocks(x, [f"dec.blk{i}" for i in range(cfg.dec_blocks)])
    surface = torch.empty(sshape, dtype=torch.float32, device="cuda")
    atmos = torch.empty(ashape, dtype=torch.float32, device="cuda")
    if host_out is None:
        decode_planes(dm.decoder(), dm.buffers(), cfg, x, surface, atmos)
        return DecodedFields(lat.valid_time, Tensor(device=surface), Tensor(device=atmos))
    main, side = torch.cuda.current_stream(), _copy_stream()
    pl = cfg.level_patch

    def on_plane(q: int) -> None:
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            if q == 0:
                hs.copy_(surface, non_blocking=True)
            else:  # level group q - 1: one contiguous run of levels per variable
                for a in range(cfg.atmos_vars):
                    ha[a, (q - 1) * pl:q * pl].copy_(atmos[a, (q - 1) * pl:q * pl], non_blocking=True)

    decode_planes(dm.decoder(), dm.buffers(), cfg, x, surface, atmos, on_plane=on_plane)
    main.wait_stream(side)  # the device buffers stay alive and the caller's synchronisation covers the copies
    out = DecodedFields(lat.valid_time, Tensor(device=surface), Tensor(device=atmos))
    out._host = host_out
    return out


def blend_latents(latents: list, weights) -> LatentState:
    """Convex combination of same-time latent states (model.py:424-449)."""
    if not latents:
        raise ConfigError("blend of zero latent states")
    t0, ext = latents[0].valid_time, latents[0].extents
    for lt in latents[1:]:
        if lt.valid_time != t0:
            raise ConfigError(f"blend of mismatched valid times {t0} and {lt.valid_time}")
        if tuple(lt.extents) != tuple(ext):
            raise ConfigError("blend of mismatched latent extents")
    w = host_array(weights, np.float64)
    if w.shape != (len(latents),):
        raise ConfigError(f"{len(latents)} states but weight shape {w.shape}")
    if (w < 0).any() or abs(w.sum() - 1.0) > 1e-12:
        raise ConfigError("blend weights must be nonnegative and sum to 1")
    out = _tokens(latents[0]) * float(w[0])
    for wi, lt in zip(w[1:], latents[1:]):
        out.add_(_tokens(lt), alpha=float(wi))
    return LatentState(Tensor(device=out), t0, ext)
