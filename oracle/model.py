"""Oracle restatement of the reference forward path in float64 numpy — TEST INFRASTRUCTURE ONLY.

Follows, function by function (paths relative to the reference's pkg/src/gridcast/):
  rotary_tables / apply_rotary   attention.py:39-92
  layernorm                      autodiff.py:400-424  (eps 1e-6, biased variance)
  gelu                           autodiff.py:372-382  (exact erf)
  natten_block                   attention.py:146-184 (explicit neighbor gather, chunked over tokens)
  attention_weights              attention.py:187-212
  conv3x3 / conv_transpose4x4    autodiff.py:585-764 via model.py:296-325 (row zero pad, col wrap)
  encode / process / decode      model.py:332-421
  greedy_plan / rollout / forecast  rollout.py:33-91
Parameters are a dict name -> float64 ndarray (anything exposing `.values` is unwrapped).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

from .grid import OracleConfigError, neighborhood, static_fields

INV_SQRT2 = 1.0 / math.sqrt(2.0)
DOWNSAMPLE_STAGES = 3


def _v(t):
    return np.asarray(getattr(t, "values", t), dtype=np.float64)


# ------------------------------------------------------------------------------------------------
# block primitives
# ------------------------------------------------------------------------------------------------
def pair_split(n_pairs: int):
    """attention.py:39-42."""
    base = n_pairs // 3
    return base, base, n_pairs - 2 * base


def axis_wavelengths(extent: int, n: int) -> np.ndarray:
    """attention.py:70-74."""
    lo, hi = 4.0, max(8.0, 2.0 * extent)
    if n == 1:
        return np.array([hi])
    return lo * (hi / lo) ** (np.arange(n) / (n - 1))


def rotary_angles(extents, head_dim: int) -> np.ndarray:
    """attention.py:48-84 — (T, head_dim//2) float64 phase angles."""
    if head_dim % 2 != 0:
        raise OracleConfigError(f"rotary head dim must be even, got {head_dim}")
    n = head_dim // 2
    if n < 3:
        raise OracleConfigError(f"head dim {head_dim} leaves fewer than one rotary pair per axis")
    pd, pr, pc = pair_split(n)
    d, h, w = extents
    di, hi, wi = np.unravel_index(np.arange(d * h * w), (d, h, w))
    ang = np.empty((d * h * w, n), dtype=np.float64)
    ang[:, :pd] = 2.0 * math.pi * di[:, None] / axis_wavelengths(d, pd)[None, :]
    ang[:, pd:pd + pr] = 2.0 * math.pi * hi[:, None] / axis_wavelengths(h, pr)[None, :]
    ang[:, pd + pr:] = 2.0 * math.pi * wi[:, None] * np.arange(1, pc + 1, dtype=np.float64)[None, :] / w
    return ang


_ROT: dict = {}
_NB: dict = {}


def rotary_tables(extents, head_dim: int):
    """Cached like the reference (attention.py:45)."""
    key = (tuple(extents), head_dim)
    if key not in _ROT:
        ang = rotary_angles(extents, head_dim)
        _ROT[key] = (np.cos(ang)[:, None, :], np.sin(ang)[:, None, :])
    return _ROT[key]


def _neighborhood(extents, window):
    """Cached like the reference (grid.py:104)."""
    key = (tuple(extents), tuple(window))
    if key not in _NB:
        _NB[key] = neighborhood(extents, window)
    return _NB[key]


def apply_rotary(x: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """attention.py:87-92 — NeoX half split over the last axis of (T, heads, dh)."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x1 * sin + x2 * cos], axis=-1)


def layernorm(x: np.ndarray, gain, bias, eps: float = 1e-6) -> np.ndarray:
    """autodiff.py:400-424."""
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=-1, keepdims=True)
    return xc / np.sqrt(var + eps) * _v(gain) + _v(bias)


def gelu(x: np.ndarray) -> np.ndarray:
    """autodiff.py:372-382 — exact erf GELU."""
    return 0.5 * x * (1.0 + erf(x * INV_SQRT2))


def _attend(q, k, v, table, scale, chunk):
    """softmax(q k^T * scale) v over each token's neighbor list, chunked over tokens."""
    t, heads, dh = q.shape
    out = np.empty_like(q)
    for s in range(0, t, chunk):
        e = min(t, s + chunk)
        idx = table[s:e]
        kn = k[idx]  # (c, K, heads, dh)
        vn = v[idx]
        sc = np.einsum("chd,ckhd->chk", q[s:e], kn) * scale
        sc = sc - sc.max(axis=-1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(axis=-1, keepdims=True)
        out[s:e] = np.einsum("chk,ckhd->chd", p, vn)
    return out


def natten_block(x: np.ndarray, params: dict, prefix: str, extents, window, heads: int,
                 chunk: int = 512) -> np.ndarray:
    """attention.py:146-184 — pre-norm neighborhood-attention block on tokens (T, dim)."""
    t, dim = x.shape
    d, h, w = extents
    if t != d * h * w:
        raise OracleConfigError(f"token count {t} != prod of extents {extents}")
    if dim % heads != 0:
        raise OracleConfigError(f"dim {dim} not divisible by heads {heads}")
    dh = dim // heads
    table = _neighborhood(extents, window)
    cos, sin = rotary_tables(extents, dh)

    def p(name):
        return _v(params[f"{prefix}.{name}"])

    hn = layernorm(x, p("ln1.gain"), p("ln1.bias"))
    q = (hn @ p("attn.wq") + p("attn.bq")).reshape(t, heads, dh)
    k = (hn @ p("attn.wk") + p("attn.bk")).reshape(t, heads, dh)
    v = (hn @ p("attn.wv") + p("attn.bv")).reshape(t, heads, dh)
    q = apply_rotary(q, cos, sin)
    k = apply_rotary(k, cos, sin)
    ctx = _attend(q, k, v, table, 1.0 / math.sqrt(dh), chunk).reshape(t, dim)
    x = x + ctx @ p("attn.wo") + p("attn.bo")
    hn2 = layernorm(x, p("ln2.gain"), p("ln2.bias"))
    mid = gelu(hn2 @ p("mlp.w1") + p("mlp.b1"))
    return x + mid @ p("mlp.w2") + p("mlp.b2")


def attention_weights(x: np.ndarray, params: dict, prefix: str, extents, window, heads: int) -> np.ndarray:
    """attention.py:187-212 — softmax weights (T, heads, K)."""
    t, dim = x.shape
    dh = dim // heads
    table = _neighborhood(extents, window)
    cos, sin = rotary_tables(extents, dh)

    def p(name):
        return _v(params[f"{prefix}.{name}"])

    hn = layernorm(x, p("ln1.gain"), p("ln1.bias"))
    q = apply_rotary((hn @ p("attn.wq") + p("attn.bq")).reshape(t, heads, dh), cos, sin)
    k = apply_rotary((hn @ p("attn.wk") + p("attn.bk")).reshape(t, heads, dh), cos, sin)
    sc = np.einsum("thd,tkhd->thk", q, k[table]) / math.sqrt(dh)
    sc = sc - sc.max(axis=-1, keepdims=True)
    e = np.exp(sc)
    return e / e.sum(axis=-1, keepdims=True)


# ------------------------------------------------------------------------------------------------
# convolutions: rows zero-padded, columns periodic (model.py:296-325, autodiff.py:585-764)
# ------------------------------------------------------------------------------------------------
def conv3x3(x: np.ndarray, w, b, stride: int = 1) -> np.ndarray:
    """(Cin, H, W) -> (Cout, Ho, Wo); taps rows {s*o-1, s*o, s*o+1} (zero outside), cols wrap."""
    w = _v(w)
    b = _v(b)
    cin, hh, ww = x.shape
    cout = w.shape[0]
    ho = (hh + 2 - 3) // stride + 1
    if ww % stride:
        raise OracleConfigError(f"conv: wrapped extent {ww} not divisible by stride {stride}")
    wo = ww // stride
    xp = np.zeros((cin, hh + 2, ww + 2), dtype=np.float64)
    xp[:, 1:-1, 1:-1] = x
    xp[:, 1:-1, 0] = x[:, :, -1]
    xp[:, 1:-1, -1] = x[:, :, 0]
    y = np.zeros((cout, ho * wo), dtype=np.float64)
    for kh in range(3):
        for kw in range(3):
            tap = xp[:, kh:kh + stride * (ho - 1) + 1:stride, kw:kw + stride * (wo - 1) + 1:stride]
            y += w[:, :, kh, kw] @ tap.reshape(cin, -1)
    return (y + b[:, None]).reshape(cout, ho, wo)


def conv_transpose4x4s2(x: np.ndarray, w, b, out_hw) -> np.ndarray:
    """Adjoint of the k=4, s=2, rows-pad-(1,1), cols-wrap conv: x[:, o] feeds rows/cols 2o-1..2o+2."""
    w = _v(w)
    b = _v(b)
    cin, h, wd = x.shape
    cout = w.shape[1]
    H, W = out_hw
    if (H + 2 - 4) // 2 + 1 != h or W // 2 != wd:
        raise OracleConfigError(f"conv_transpose: geometry {out_hw} -> {(h, wd)} mismatch")
    y = np.zeros((cout, H + 2, W), dtype=np.float64)  # rows offset by 1 (pad), cols modulo W
    xf = x.reshape(cin, -1)
    cols = np.arange(wd)
    for kh in range(4):
        rows = 2 * np.arange(h) + kh  # padded row index (2o + kh - 1) + 1
        for kw in range(4):
            contrib = (w[:, :, kh, kw].T @ xf).reshape(cout, h, wd)
            cidx = (2 * cols + kw - 1) % W
            y[:, rows[:, None], cidx[None, :]] += contrib
    return y[:, 1:-1] + b[:, None, None]


# ------------------------------------------------------------------------------------------------
# model (model.py:332-421)
# ------------------------------------------------------------------------------------------------
def _conv(x, params, name, stride=1):
    return conv3x3(x, params[name + ".w"], params[name + ".b"], stride)


def _res_block(x, params, name):
    return x + _conv(gelu(_conv(x, params, name + ".conv1")), params, name + ".conv2")


def pyramid_down(x, params, prefix):
    for i in range(DOWNSAMPLE_STAGES):
        x = _conv(x, params, f"{prefix}.stage{i}.down", stride=2)
        x = _res_block(x, params, f"{prefix}.stage{i}.res0")
        x = _res_block(x, params, f"{prefix}.stage{i}.res1")
    return x


def pyramid_up(x, params, out_shapes):
    for i in range(DOWNSAMPLE_STAGES):
        x = conv_transpose4x4s2(x, params[f"dec.stage{i}.up.w"], params[f"dec.stage{i}.up.b"], out_shapes[i])
        x = _res_block(x, params, f"dec.stage{i}.res0")
        x = _res_block(x, params, f"dec.stage{i}.res1")
    return x


def encode(surface: np.ndarray, atmos: np.ndarray, params: dict, cfg, prefix: str = "enc") -> np.ndarray:
    """model.py:363-390 -> tokens (T, hidden)."""
    g = cfg.grid
    stat = static_fields(g.rows, g.cols, g.north_lat, g.lat_step, g.lon_step)
    planes = [_conv(np.concatenate([surface, stat], axis=0), params, f"{prefix}.stem_sfc")]
    a, lv, hh, ww = atmos.shape
    grp = lv // cfg.level_patch
    folded = atmos.reshape(a, grp, cfg.level_patch, hh, ww).transpose(1, 0, 2, 3, 4)
    for j in range(grp):
        planes.append(_conv(folded[j].reshape(a * cfg.level_patch, hh, ww), params, f"{prefix}.stem_atm"))
    planes = [pyramid_down(pl, params, prefix) for pl in planes]
    tokens = np.stack(planes, axis=0).transpose(0, 2, 3, 1).reshape(-1, cfg.hidden)
    ext = cfg.latent_extents
    for i in range(cfg.enc_blocks):
        tokens = natten_block(tokens, params, f"{prefix}.blk{i}", ext, cfg.window, cfg.heads)
    return tokens


def process(tokens: np.ndarray, params: dict, cfg, horizon: int) -> np.ndarray:
    """model.py:393-405."""
    for i in range(cfg.proc_blocks):
        tokens = natten_block(tokens, params, f"proc{horizon}.blk{i}", cfg.latent_extents, cfg.window, cfg.heads)
    return tokens


def decode(tokens: np.ndarray, params: dict, cfg):
    """model.py:408-421 -> (surface (surface_out, H, W), atmos (A, L, H, W))."""
    ext = cfg.latent_extents
    for i in range(cfg.dec_blocks):
        tokens = natten_block(tokens, params, f"dec.blk{i}", ext, cfg.window, cfg.heads)
    g = cfg.grid
    up = [(g.rows // 4, g.cols // 4), (g.rows // 2, g.cols // 2), (g.rows, g.cols)]
    d, hh, ww = ext
    planes = tokens.reshape(d, hh, ww, cfg.hidden).transpose(0, 3, 1, 2)
    full = [pyramid_up(planes[j], params, up) for j in range(d)]
    surface = _conv(full[0], params, "dec.head_sfc")
    atm = np.stack([_conv(pl, params, "dec.head_atm") for pl in full[1:]], axis=0)  # (G, A*P, H, W)
    atm = atm.reshape(d - 1, cfg.atmos_vars, cfg.level_patch, g.rows, g.cols).transpose(1, 0, 2, 3, 4)
    return surface, atm.reshape(cfg.atmos_vars, (d - 1) * cfg.level_patch, g.rows, g.cols)


def greedy_plan(dt: int, max_dt: int = 336):
    """rollout.py:33-41."""
    if not isinstance(dt, int) or isinstance(dt, bool):
        raise OracleConfigError(f"dt must be an integer hour count, got {dt!r}")
    if dt < 0 or dt > max_dt:
        raise OracleConfigError(f"dt {dt} outside [0, {max_dt}]")
    return (6,) * (dt // 6) + (1,) * (dt % 6)


def rollout(tokens: np.ndarray, plan, params: dict, cfg) -> np.ndarray:
    """rollout.py:56-81 (latent only)."""
    for hz in plan:
        tokens = process(tokens, params, cfg, hz)
    return tokens


def forecast(surface, atmos, dt: int, params: dict, cfg):
    """rollout.py:84-91."""
    tokens = encode(surface, atmos, params, cfg)
    tokens = rollout(tokens, greedy_plan(dt, cfg.max_dt), params, cfg)
    return decode(tokens, params, cfg)


def block_flops(tokens: int, dim: int, keys: int) -> float:
    """Algorithmic FLOPs of one block: 24 T D^2 (QKV, O, 4x MLP) + 4 T K D (q k^T and P V)."""
    return 24.0 * tokens * dim * dim + 4.0 * tokens * keys * dim
