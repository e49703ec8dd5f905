"""Device-resident neighborhood-attention block: weight layout, rotary tables, forward chain.

One block (attention.py:146-184) is seven launches on one stream:
  LN1 -> [QKV GEMM + bias + rotary] -> [fused NA] -> [O-proj GEMM + bias + residual]
      -> LN2 -> [W1 GEMM + bias + GELU] -> [W2 GEMM + bias + residual]
The residual stream x stays fp32 (T, hidden) in HBM; GEMM operands are bf16, accumulation fp32 in TMEM.

Weight layout (built once per parameter set, from the reference's (in, out) float64 matrices):
  * every GEMM weight is stored (out, in) = K-major bf16 so both UMMA operands are K-major SW128 tiles;
  * K and N are padded to the kernels' granularity with zero rows/columns (exact);
  * heads are padded to dhp in {64, 128}; within a q/k head the rotary pair (j, j + dh/2) of the reference
    is placed at the adjacent columns (2j, 2j + 1) — the same permutation on q and k leaves q.k unchanged.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, ops
from .errors import ConfigError
from .params import block_param_names
from .tensor import host_values


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def head_pad(dh: int) -> int:
    if dh <= 64:
        return 64
    if dh <= 128:
        return 128
    raise ConfigError(f"head dim {dh} > 128 is not supported by the fused attention kernel")


# ------------------------------------------------------------------------------------------------
# rotary phases (attention.py:39-84), as per-axis fp32 tables for the QKV epilogue
# ------------------------------------------------------------------------------------------------
def pair_split(n_pairs: int) -> tuple[int, int, int]:
    base = n_pairs // 3
    return base, base, n_pairs - 2 * base


def _wavelengths(extent: int, n: int) -> np.ndarray:
    lo, hi = 4.0, max(8.0, 2.0 * extent)
    if n == 1:
        return np.array([hi])
    return lo * (hi / lo) ** (np.arange(n) / (n - 1))


def rope_axis_tables(extents, head_dim: int):
    """(cos, sin) float32 arrays of shape (3, emax, 64): axis 0 depth, 1 row, 2 col; unused = (1, 0)."""
    if head_dim % 2:
        raise ConfigError(f"rotary head dim must be even, got {head_dim}")
    n = head_dim // 2
    if n < 3:
        raise ConfigError(f"head dim {head_dim} leaves fewer than one rotary pair per axis")
    pd, pr, pc = pair_split(n)
    d, h, w = (int(e) for e in extents)
    emax = max(d, h, w)
    ang = np.zeros((3, emax, 64), dtype=np.float64)
    use = np.zeros((3, 64), dtype=bool)
    ang[0, :d, :pd] = 2.0 * math.pi * np.arange(d)[:, None] / _wavelengths(d, pd)[None, :]
    use[0, :pd] = True
    ang[1, :h, pd:pd + pr] = 2.0 * math.pi * np.arange(h)[:, None] / _wavelengths(h, pr)[None, :]
    use[1, pd:pd + pr] = True
    ang[2, :w, pd + pr:n] = 2.0 * math.pi * np.arange(w)[:, None] * np.arange(1, pc + 1)[None, :] / w
    use[2, pd + pr:n] = True
    cos = np.where(use[:, None, :], np.cos(ang), 1.0).astype(np.float32)
    sin = np.where(use[:, None, :], np.sin(ang), 0.0).astype(np.float32)
    return cos, sin, pd, pr, emax


# ------------------------------------------------------------------------------------------------
# weights
# ------------------------------------------------------------------------------------------------
@dataclass
class BlockWeights:
    """Device layout of one block's parameters (see prepare_block)."""
    hidden: int
    heads: int
    dh: int
    dhp: int
    kp: int        # padded hidden as a GEMM K (LN output pitch)
    np_: int       # padded hidden as a GEMM N
    nm: int        # padded MLP width
    ln1_g: torch.Tensor
    ln1_b: torch.Tensor
    w_qkv: torch.Tensor
    b_qkv: torch.Tensor
    w_o: torch.Tensor
    b_o: torch.Tensor
    ln2_g: torch.Tensor
    ln2_b: torch.Tensor
    w_1: torch.Tensor
    b_1: torch.Tensor
    w_2: torch.Tensor
    b_2: torch.Tensor
    # LayerNorm folded into the QKV / W1 GEMMs (wm3_ln_fold_t): gain-scaled weights, their column sums and the
    # shifted biases; None = separate LayerNorm launches (the default; WM3_LN_FOLD=1 folds)
    w_qkv_f: torch.Tensor | None = None
    c_qkv: torch.Tensor | None = None
    d_qkv: torch.Tensor | None = None
    w_1_f: torch.Tensor | None = None
    c_1: torch.Tensor | None = None
    d_1: torch.Tensor | None = None

    @property
    def folded(self) -> bool:
        return self.w_qkv_f is not None

    @property
    def ln_parts(self) -> int:
        """Partial-sum pairs per row the residual GEMMs write (gemm.cu: 2 epilogue groups per column tile)."""
        bn = 256 if self.np_ >= 256 else 128
        return 2 * ((self.np_ + bn - 1) // bn)

    def native(self) -> "_lib.BlockWeightsT":
        """wm3_block_weights_t view of these tensors (cached; the tensors stay owned by this object)."""
        nat = self.__dict__.get("_native")
        if nat is None:
            fold = [(t.data_ptr() if t is not None else None)
                    for t in (self.w_qkv_f, self.c_qkv, self.d_qkv, self.w_1_f, self.c_1, self.d_1)]
            nat = _lib.BlockWeightsT(*(t.data_ptr() for t in (self.ln1_g, self.ln1_b, self.w_qkv, self.b_qkv, self.w_o,
                                                              self.b_o, self.ln2_g, self.ln2_b, self.w_1, self.b_1,
                                                              self.w_2, self.b_2)),
                                     self.hidden, self.heads, self.dh, self.dhp, self.kp, self.np_, self.nm, *fold)
            self.__dict__["_native"] = nat
        return nat


def _qk_perm(heads: int, dh: int, dhp: int) -> np.ndarray:
    """Padded column -> reference column (or -1) for a q/k section.

    Rotary pair j of the reference, columns (j, j + dh/2) (attention.py:87-92), lands on the adjacent
    columns (2j, 2j + 1) so every 64-column epilogue chunk holds whole pairs.
    """
    m = np.full(heads * dhp, -1, dtype=np.int64)
    half = dh // 2
    for hh in range(heads):
        for j in range(half):
            m[hh * dhp + 2 * j] = hh * dh + j
            m[hh * dhp + 2 * j + 1] = hh * dh + half + j
    return m


def _v_perm(heads: int, dh: int, dhp: int) -> np.ndarray:
    m = np.full(heads * dhp, -1, dtype=np.int64)
    for hh in range(heads):
        m[hh * dhp: hh * dhp + dh] = hh * dh + np.arange(dh)
    return m


def _gather_cols(w: np.ndarray, perm: np.ndarray) -> np.ndarray:
    """w (in, out) -> (in, len(perm)) picking columns perm (-1 -> zero)."""
    out = np.zeros((w.shape[0], perm.size), dtype=np.float64)
    ok = perm >= 0
    out[:, ok] = w[:, perm[ok]]
    return out


def _kmajor_bf16(w_in_out: np.ndarray, n_pad: int, k_pad: int, device) -> torch.Tensor:
    """(in, out) float64 -> (n_pad, k_pad) bf16, zero padded."""
    k, n = w_in_out.shape
    buf = np.zeros((n_pad, k_pad), dtype=np.float32)
    buf[:n, :k] = w_in_out.T
    return torch.from_numpy(buf).to(device=device, dtype=_lib.ELEM)


def _vec(v: np.ndarray, n_pad: int, device) -> torch.Tensor:
    buf = np.zeros(n_pad, dtype=np.float32)
    buf[: v.size] = v
    return torch.from_numpy(buf).to(device)


def _fold_ln(w_in_out: np.ndarray, bias: np.ndarray, gain: np.ndarray, beta: np.ndarray, n_pad: int, k_pad: int,
             device):
    """LayerNorm folded into the GEMM that follows it: LN(x) W + b = rstd (x W') - rstd mean c + d with
    W' = diag(gain) W (stored fp16), c = column sums of the stored fp16 W' (so the mean term cancels exactly what
    the tensor cores accumulate), d = b + beta W."""
    k = w_in_out.shape[0]
    wf = _kmajor_bf16(w_in_out * gain[:k, None], n_pad, k_pad, device)
    c = wf.double().cpu().numpy().sum(axis=1)
    d = np.zeros(n_pad, dtype=np.float64)
    d[: w_in_out.shape[1]] = bias + beta[:k] @ w_in_out
    return wf, _vec(c, n_pad, device), _vec(d, n_pad, device)


def ln_fold_enabled() -> bool:
    """WM3_LN_FOLD=1 selects the folded LayerNorm (no LayerNorm launches; two tiny row-statistics launches).
    Off by default: measured in-block on one B200 the epilogue work it adds costs about what the two LayerNorm
    launches cost (2.127 vs 2.111 ms per block)."""
    return os.environ.get("WM3_LN_FOLD", "0") == "1"


def prepare_block(params: dict, prefix: str, heads: int, device="cuda") -> BlockWeights:
    names = block_param_names(prefix)
    missing = [n for n in names if n not in params]
    if missing:
        raise ConfigError(f"missing block parameters {missing[:3]}...")
    p = {n[len(prefix) + 1:]: host_values(params[n]) for n in names}
    hidden = p["ln1.gain"].shape[0]
    if hidden % heads:
        raise ConfigError(f"dim {hidden} not divisible by heads {heads}")
    dh = hidden // heads
    dhp = head_pad(dh)
    kp = round_up(hidden, 64)
    np_ = round_up(hidden, 32)
    nm = round_up(p["mlp.w1"].shape[1], 64)
    qk = _qk_perm(heads, dh, dhp)
    vv = _v_perm(heads, dh, dhp)
    w_qkv = np.concatenate([_gather_cols(p["attn.wq"], qk), _gather_cols(p["attn.wk"], qk),
                            _gather_cols(p["attn.wv"], vv)], axis=1)
    b_qkv = np.concatenate([_gather_cols(p["attn.bq"][None], qk)[0], _gather_cols(p["attn.bk"][None], qk)[0],
                            _gather_cols(p["attn.bv"][None], vv)[0]])
    # O-proj input rows follow the padded ctx layout (v order)
    wo = np.zeros((heads * dhp, hidden), dtype=np.float64)
    ok = vv >= 0
    wo[ok] = p["attn.wo"][vv[ok]]
    fold = {}
    if ln_fold_enabled():
        fold["w_qkv_f"], fold["c_qkv"], fold["d_qkv"] = _fold_ln(w_qkv, b_qkv, p["ln1.gain"], p["ln1.bias"],
                                                                 3 * heads * dhp, kp, device)
        fold["w_1_f"], fold["c_1"], fold["d_1"] = _fold_ln(p["mlp.w1"], p["mlp.b1"], p["ln2.gain"], p["ln2.bias"],
                                                           nm, kp, device)
    return BlockWeights(
        hidden=hidden, heads=heads, dh=dh, dhp=dhp, kp=kp, np_=np_, nm=nm,
        ln1_g=_vec(p["ln1.gain"], hidden, device), ln1_b=_vec(p["ln1.bias"], hidden, device),
        w_qkv=_kmajor_bf16(w_qkv, 3 * heads * dhp, kp, device), b_qkv=_vec(b_qkv, 3 * heads * dhp, device),
        w_o=_kmajor_bf16(wo, np_, heads * dhp, device), b_o=_vec(p["attn.bo"], np_, device),
        ln2_g=_vec(p["ln2.gain"], hidden, device), ln2_b=_vec(p["ln2.bias"], hidden, device),
        w_1=_kmajor_bf16(p["mlp.w1"], nm, kp, device), b_1=_vec(p["mlp.b1"], nm, device),
        w_2=_kmajor_bf16(p["mlp.w2"], np_, nm, device), b_2=_vec(p["mlp.b2"], np_, device), **fold,
    )


# ------------------------------------------------------------------------------------------------
# forward
# ------------------------------------------------------------------------------------------------
class RopeTables:
    """Device copy of the per-axis rotary tables for one (global extents, dh), plus the ctypes struct."""

    def __init__(self, extents, dh: int, device="cuda"):
        cos, sin, pd, pr, emax = rope_axis_tables(extents, dh)
        self.cos = torch.from_numpy(cos).to(device)
        self.sin = torch.from_numpy(sin).to(device)
        self.pd, self.pr, self.emax = pd, pr, emax
        self.extents = tuple(int(e) for e in extents)
        self._bands: dict = {}

    def band_tables(self, local_extents, row0: int):
        """(dr, col) device tables of wm3_rope_t for a band of `local_extents` starting at global row row0:
        dr [d * rows][2][64] (depth / row pairs of each (plane, band row); column pairs (1, 0)) and col
        [2][64][cols] pair-major (column pairs of each column; other pairs (1, 0))."""
        d, h, w = (int(e) for e in local_extents)
        key = (d, h, w, int(row0))
        hit = self._bands.get(key)
        if hit is None:
            dev = self.cos.device
            pair = torch.arange(64, device=dev)
            split = self.pd + self.pr
            dd = torch.arange(d, device=dev).view(d, 1).expand(d, h).reshape(-1)
            rr = (torch.arange(h, device=dev) + int(row0)).view(1, h).expand(d, h).reshape(-1)
            axis = torch.where(pair < self.pd, 0, torch.where(pair < split, 1, 2))           # (64,)
            coord = torch.where(axis == 0, dd[:, None], rr[:, None])                          # (d*h, 64)
            coord = torch.where(axis[None, :] == 2, 0, coord)
            ax = axis.clamp(max=1).expand_as(coord)
            is_col = (axis == 2)[None, :]
            c_dr = torch.where(is_col, 1.0, self.cos[ax, coord, pair.expand_as(coord)])
            s_dr = torch.where(is_col, 0.0, self.sin[ax, coord, pair.expand_as(coord)])
            dr = torch.stack([c_dr, s_dr], 1).contiguous()                                    # (d*h, 2, 64)
            cc = torch.arange(w, device=dev)
            c_col = torch.where(is_col.T, self.cos[2][cc][:, pair].T, 1.0)                    # (64, w)
            s_col = torch.where(is_col.T, self.sin[2][cc][:, pair].T, 0.0)
            col = torch.stack([c_col, s_col], 0).contiguous()                                  # (2, 64, w)
            hit = (dr, col, split)
            self._bands[key] = hit
        return hit

    def struct(self, local_extents, row0: int, heads: int, dhp: int) -> _lib.RopeT:
        d, h, w = (int(e) for e in local_extents)
        dr, col, split = self.band_tables(local_extents, row0)
        return _lib.RopeT(dr.data_ptr(), col.data_ptr(), heads, dhp, h, w, d * h * w, split)


class Workspace:
    """Scratch activations for one (band geometry, block shape); reused across blocks and steps.

    qkv lives in the padded K/V grid of ops.KVGrid (wrap columns + latitude-band halo rows)."""

    def __init__(self, grid: "ops.KVGrid", bw: BlockWeights, device="cuda"):
        self.grid = grid
        tokens = grid.batch * grid.depth * grid.rows * grid.cols
        self.tokens = tokens
        self.hn = torch.zeros((tokens, bw.kp), dtype=_lib.ELEM, device=device)  # pad columns stay zero
        self.qkv = torch.zeros((grid.tokens, 3 * bw.heads * bw.dhp), dtype=_lib.ELEM, device=device)
        self.ctx = torch.empty((tokens, bw.heads * bw.dhp), dtype=_lib.ELEM, device=device)
        self.mid = torch.empty((tokens, bw.nm), dtype=_lib.ELEM, device=device)
        # LayerNorm-fold row statistics ([tokens][WM3_LN_SLOTS] (sum, sum of squares) pairs)
        self.stats = torch.zeros((tokens, 2 * _lib.LN_SLOTS), dtype=torch.float32, device=device)
        self.row_stats = torch.zeros((tokens, 2), dtype=torch.float32, device=device)
        self._native = _lib.BlockWsT(self.hn.data_ptr(), self.qkv.data_ptr(), self.ctx.data_ptr(),
                                     self.mid.data_ptr(), self.stats.data_ptr(), self.row_stats.data_ptr())

    def native(self) -> "_lib.BlockWsT":
        return self._native


def block_forward(x: torch.Tensor, bw: BlockWeights, ws: Workspace, rope: RopeTables, extents, window,
                  row0: int = 0, rows_global: int | None = None, halo_exchange=None, mark=None,
                  prepped: bool = False) -> None:
    """In-place x (T, hidden) fp32 <- natten_block(x) on the current stream.

    With a batched workspace (ws.grid.batch = B ensemble members) x is (B * T, hidden), member-major; the
    members never see each other (per-token ops are row-parallel, attention windows stay in a member).

    extents are the local (band) token extents; row0 / rows_global place the band in the global grid
    (rotary phases and window bumps use global rows).  halo_exchange(qkv, grid), when given, fills the halo
    rows of the padded K/V grid from the neighbouring bands between the QKV GEMM and the attention kernel.
    Launches with the folded LayerNorm (bw.folded): [LN-fold prep unless `prepped`], QKV+rotary GEMM, NA,
    O-proj+residual GEMM (+ fp16 copy and row statistics of x), W1+GELU GEMM, W2+residual GEMM (+ the same for
    the next block, which may then pass prepped=True); otherwise LN1, QKV, NA, O-proj, LN2, W1, W2.
    mark(i), when given, is called before launch slot i (0..6: LN1 / prep, QKV, NA, O-proj, LN2, W1, W2) and once
    more after the last (profiling: CUDA events; the folded path leaves slot 4 empty).
    """
    L = _lib
    g = ws.grid
    d, h, w = (int(e) for e in extents)
    rg = int(rows_global if rows_global is not None else h)
    if mark is None and halo_exchange is None:
        # the whole block in one library call (wm3_block_fwd: the launches are issued by the C++ host code)
        import ctypes
        rs = rope.struct(extents, row0, bw.heads, bw.dhp)
        geom = L.BlockGeomT(g.batch, d, h, w, rg, int(row0), g.halo_lo, g.halo_hi, *(int(v) for v in window),
                            int(bool(prepped)))
        L.check(L.lib().wm3_block_fwd(x.data_ptr(), ctypes.byref(bw.native()), ctypes.byref(ws.native()),
                                      ctypes.byref(geom), ctypes.byref(rs), L.stream_ptr()), "wm3_block_fwd")
        return
    mk = mark if mark is not None else (lambda i: None)
    rs = rope.struct(extents, row0, bw.heads, bw.dhp)
    if bw.folded:
        parts = bw.ln_parts
        cons_qkv = ops.ln_fold_consumer(ws.row_stats, bw.c_qkv)
        cons_1 = ops.ln_fold_consumer(ws.row_stats, bw.c_1)
        prod = ops.ln_fold_producer(ws.hn, ws.stats)
        mk(0)
        if not prepped:
            ops.ln_fold_prep(x, bw.hidden, ws.hn, ws.row_stats)
        mk(1)
        ops.linear_grid(ws.hn, bw.w_qkv_f, L.WM3_EPI_QKV_ROPE, bw.d_qkv, ws.qkv, g, rope=rs, fold=cons_qkv)
        if halo_exchange is not None:
            halo_exchange(ws.qkv, g)
        mk(2)
        ops.natten(ws.qkv, g, bw.heads, bw.dhp, bw.dh, window, out=ws.ctx, rows_global=rows_global, row0=row0)
        mk(3)
        ops.linear(ws.ctx, bw.w_o, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=x, n_valid=bw.hidden, fold=prod)
        mk(4)
        ops.ln_fold_finalize(ws.stats, parts, bw.hidden, ws.row_stats)
        mk(5)
        ops.linear(ws.hn, bw.w_1_f, L.WM3_EPI_BIAS_GELU_BF16, bias=bw.d_1, out=ws.mid, fold=cons_1)
        mk(6)
        ops.linear(ws.mid, bw.w_2, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_2, out=x, n_valid=bw.hidden, fold=prod)
        ops.ln_fold_finalize(ws.stats, parts, bw.hidden, ws.row_stats)  # for the next block (counted in W2's slot)
        mk(7)
        return
    mk(0)
    ops.layernorm_bf16(x, bw.ln1_g, bw.ln1_b, out=ws.hn)
    mk(1)
    ops.linear_grid(ws.hn, bw.w_qkv, L.WM3_EPI_QKV_ROPE, bw.b_qkv, ws.qkv, g, rope=rs)
    if halo_exchange is not None:
        halo_exchange(ws.qkv, g)
    mk(2)
    ops.natten(ws.qkv, g, bw.heads, bw.dhp, bw.dh, window, out=ws.ctx, rows_global=rows_global, row0=row0)
    mk(3)
    ops.linear(ws.ctx, bw.w_o, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=x, n_valid=bw.hidden)
    mk(4)
    ops.layernorm_bf16(x, bw.ln2_g, bw.ln2_b, out=ws.hn)
    mk(5)
    ops.linear(ws.hn, bw.w_1, L.WM3_EPI_BIAS_GELU_BF16, bias=bw.b_1, out=ws.mid)
    mk(6)
    ops.linear(ws.mid, bw.w_2, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_2, out=x, n_valid=bw.hidden)
    mk(7)
