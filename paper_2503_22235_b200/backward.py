"""Reverse mode of the B200 processor block: the vector-Jacobian product of natten_block.

`block_vjp(x, params, prefix, extents, window, heads, gy)` returns (gx, {parameter name: gradient}) in the
reference's layouts (float64 numpy, parameter shapes of attention.py:105-139), i.e. what the reference tape's
rules for the block's primitives accumulate (autodiff.py:350-424, 516-533; attention.py:146-184).

Device chain (one stream; every launch a libwm3 kernel):
  forward recompute from x (the tape saves only the block input, like a checkpointed segment,
  autodiff.py:893-924): LN1, QKV+rotary GEMM, fused NA, O-proj, LN2, W1 pre-activation (fp32) and GELU output
  backward: W2 (dW2 = gy^T mid, g_mid = gy W2) -> GELU' -> W1 -> LN2 backward (+ gy) -> O-proj -> attention
  backward (query side: recomputed softmax, dS; key side: the inverse neighbor list, deterministic) -> rotary
  transpose -> QKV -> LN1 backward (+ gx1)
Weight and input gradients are tcgen05 GEMMs (wm3_linear) on 16-bit operands: gradients enter them scaled by a
per-tensor power of two (wm3_bw_amax / wm3_bw_cast), activations enter transposed (token axis = GEMM K), and the
fp32 results are unscaled by their consumers.  All summations run in fixed orders, so the same inputs give
bitwise the same gradients (checkpoint / offload parity, verify.py:73-113).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib, ops
from ._lib import check, ptr, stream_ptr
from .blocks import _qk_perm, _v_perm
from .params import block_param_names
from .runtime import CACHE

LN_EPS = 1e-6


def _r8(n: int) -> int:
    return (n + 7) // 8 * 8


class _Scale:
    """A device float-bits cell holding max |g| of one gradient tensor (the power-of-two operand scale)."""

    def __init__(self, dev):
        self.bits = torch.zeros(1, dtype=torch.int32, device=dev)

    def ptr(self):
        return self.bits.data_ptr()

    def value(self) -> float:
        amax = float(self.bits.view(torch.float32).item())
        if not amax > 0.0 or not math.isfinite(amax):
            return 1.0
        return 2.0 ** (14 - math.ceil(math.log2(amax)))


def _amax(g: torch.Tensor, rows: int, cols: int) -> _Scale:
    s = _Scale(g.device)
    check(_lib.lib().wm3_bw_amax(ptr(g), rows, cols, g.stride(0), s.ptr(), stream_ptr()), "wm3_bw_amax")
    return s


def _cast(src: torch.Tensor, rows: int, cols: int, ldd: int, transpose: bool = False,
          scale: _Scale | None = None) -> torch.Tensor:
    """16-bit operand copy of src[:rows, :cols] (times the scale), row-major [rows][ldd] or transposed
    [cols][ldd], zero padded."""
    f32 = src.dtype == torch.float32
    out = torch.empty(((cols if transpose else rows), ldd), dtype=_lib.ELEM, device=src.device)
    check(_lib.lib().wm3_bw_cast(ptr(src), int(f32), rows, cols, src.stride(0), ptr(out), ldd, int(transpose),
                                 None if scale is None else scale.ptr(), stream_ptr()), "wm3_bw_cast")
    return out


def _colsum(src: torch.Tensor, rows: int, cols: int, src2: torch.Tensor | None = None,
            scale: _Scale | None = None) -> torch.Tensor:
    chunks = (rows + 255) // 256
    partial = torch.empty((chunks, cols), dtype=torch.float32, device=src.device)
    out = torch.empty(cols, dtype=torch.float32, device=src.device)
    check(_lib.lib().wm3_bw_colsum(ptr(src), ptr(src2), rows, cols, src.stride(0),
                                   None if scale is None else scale.ptr(), ptr(partial), ptr(out), stream_ptr()),
          "wm3_bw_colsum")
    return out


def _gemm(a: torch.Tensor, b: torch.Tensor, m: int, n: int, k: int) -> torch.Tensor:
    """fp32 C[m][n] = A[m][:k] . B[n][:k]^T on the tcgen05 GEMM (raw accumulators, scaled operands)."""
    out = torch.empty((m, n), dtype=torch.float32, device=a.device)
    check(_lib.lib().wm3_linear(ptr(a), a.stride(0), ptr(b), b.stride(0), m, n, k, _lib.WM3_EPI_F32, ptr(out),
                                out.stride(0), n, None, None, stream_ptr()), "wm3_linear")
    return out


class _InverseNeighbors:
    """Key-side traversal of the window table: for each key token the (query, slot) pairs whose window holds it,
    sorted by query (grid.py:124-127 K order), as CSR on the device; with the (T, K) table itself."""

    _cache: dict = {}

    @classmethod
    def get(cls, extents, window):
        key = (tuple(extents), tuple(window), torch.cuda.current_device())
        hit = cls._cache.get(key)
        if hit is None:
            nbr = ops.neighbor_table(extents, window)
            tab = nbr.cpu().numpy()
            t_count, k_count = tab.shape
            order = np.argsort(tab.ravel(), kind="stable")  # by key, then (t, k) in row-major order
            counts = np.bincount(tab.ravel(), minlength=t_count)
            off = np.zeros(t_count + 1, dtype=np.int32)
            np.cumsum(counts, out=off[1:])
            ent = np.stack([order // k_count, order % k_count], axis=1).astype(np.int32)
            hit = (nbr, torch.from_numpy(off).cuda(), torch.from_numpy(np.ascontiguousarray(ent)).cuda(), k_count)
            cls._cache[key] = hit
        return hit


def _rope_pair_tables(extents, dh: int, dhp: int, dev) -> tuple[torch.Tensor, torch.Tensor]:
    """cos / sin (T, dhp / 2) of the interleaved pairs (pair j = reference columns (j, j + dh/2), attention.py:48-92);
    padding pairs are the identity."""
    from .attention import rotary_tables
    cos, sin = rotary_tables(extents, dh)  # (T, 1, dh / 2) float64
    t = cos.shape[0]
    c = np.ones((t, dhp // 2), dtype=np.float32)
    s = np.zeros((t, dhp // 2), dtype=np.float32)
    c[:, :dh // 2] = cos[:, 0]
    s[:, :dh // 2] = sin[:, 0]
    return torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev)


def _transposed_weights(bw) -> dict:
    """K-major copies of the block's weights for the input-gradient GEMMs (dX = dY W), cached on the weights."""
    t = bw.__dict__.get("_transposed")
    if t is None:
        t = {}
        for name, w in (("w_qkv", bw.w_qkv), ("w_o", bw.w_o), ("w_1", bw.w_1), ("w_2", bw.w_2)):
            n, k = w.shape
            t[name] = _cast(w, n, k, _r8(n), transpose=True)
        bw.__dict__["_transposed"] = t
    return t


def block_vjp(x, params: dict, prefix: str, extents, window, heads: int, gy):
    """(gx, grads) of y = natten_block(x) for the output gradient gy; numpy float64 in the reference layouts."""
    from .attention import to_device_f32, validate_block_args
    extents = tuple(int(e) for e in extents)
    window = tuple(int(w) for w in window)
    xd = to_device_f32(x)
    T, D = xd.shape
    dh = validate_block_args((T, D), extents, window, heads)
    bw = CACHE.block(params, prefix, heads)
    dev = xd.device
    dhp, hd, kp, np_, nm = bw.dhp, bw.heads * bw.dhp, bw.kp, bw.np_, bw.nm
    Tp = _r8(T)
    L = _lib
    wt = _transposed_weights(bw)
    rope = CACHE.rope(extents, dh)

    # ---- forward recompute (the kernels of the block forward, keeping the intermediates) ----
    hn = ops.layernorm_bf16(xd, bw.ln1_g, bw.ln1_b, ldo=kp)
    grid = ops.KVGrid(extents, window)
    qkv = torch.zeros((grid.tokens, 3 * hd), dtype=L.ELEM, device=dev)
    ops.linear_grid(hn, bw.w_qkv, L.WM3_EPI_QKV_ROPE, bw.b_qkv, qkv, grid, rope=rope.struct(extents, 0, heads, dhp))
    ctx = ops.natten(qkv, grid, heads, dhp, dh, window)
    x1 = xd.clone()
    ops.linear(ctx, bw.w_o, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=x1, n_valid=D)
    hn2 = ops.layernorm_bf16(x1, bw.ln2_g, bw.ln2_b, ldo=kp)
    a0 = _gemm(hn2, bw.w_1, T, nm, kp)                                   # W1 pre-activation without bias
    mid = ops.linear(hn2, bw.w_1, L.WM3_EPI_BIAS_GELU_BF16, bias=bw.b_1)  # GELU output as the forward stores it

    # ---- W2 ----
    gyd = to_device_f32(gy)
    s1 = _amax(gyd, T, D)
    gyh = _cast(gyd, T, D, np_, scale=s1)
    gyT = _cast(gyd, T, D, Tp, transpose=True, scale=s1)
    dw2 = _gemm(gyT, _cast(mid, T, nm, Tp, transpose=True), D, nm, T)   # (D, nm), x s1
    db2 = _colsum(gyd, T, D)
    g_mid = _gemm(gyh, wt["w_2"], T, nm, np_)                           # x s1
    # ---- GELU' and W1 ----
    g_a = torch.empty((T, nm), dtype=torch.float32, device=dev)
    check(L.lib().wm3_bw_gelu(ptr(g_mid), nm, ptr(a0), nm, ptr(bw.b_1), T, nm, s1.ptr(), ptr(g_a), nm, stream_ptr()),
          "wm3_bw_gelu")
    s2 = _amax(g_a, T, nm)
    dw1 = _gemm(_cast(g_a, T, nm, Tp, transpose=True, scale=s2), _cast(hn2, T, kp, Tp, transpose=True), nm, kp, T)
    db1 = _colsum(g_a, T, nm)
    g_hn2 = _gemm(_cast(g_a, T, nm, nm, scale=s2), wt["w_1"], T, kp, nm)   # x s2
    # ---- LN2 (+ the residual path gy) ----
    gx1 = torch.empty((T, D), dtype=torch.float32, device=dev)
    gxh2 = torch.empty_like(gx1)
    gsc2 = torch.empty_like(gx1)
    check(L.lib().wm3_bw_layernorm(ptr(x1), D, T, D, LN_EPS, ptr(bw.ln2_g), ptr(g_hn2), kp, s2.ptr(), ptr(gyd),
                                   ptr(gx1), ptr(gxh2), ptr(gsc2), stream_ptr()), "wm3_bw_layernorm")
    dln2_g = _colsum(gxh2, T, D)
    dln2_b = _colsum(gsc2, T, D)
    # ---- O-proj ----
    s3 = _amax(gx1, T, D)
    dwo = _gemm(_cast(gx1, T, D, Tp, transpose=True, scale=s3), _cast(ctx, T, hd, Tp, transpose=True), D, hd, T)
    dbo = _colsum(gx1, T, D)
    g_ctx = _gemm(_cast(gx1, T, D, np_, scale=s3), wt["w_o"], T, hd, np_)  # x s3
    # ---- attention (query and key sides) and the rotary transpose ----
    nbr, inv_off, inv_ent, K = _InverseNeighbors.get(extents, window)
    P = torch.empty((T, heads, K), dtype=torch.float32, device=dev)
    dS = torch.empty_like(P)
    work = torch.empty((T, heads, 2 * K), dtype=torch.float32, device=dev)
    g_qkv = torch.zeros((T, 3 * hd), dtype=torch.float32, device=dev)
    check(L.lib().wm3_bw_natten(ptr(qkv), 3 * hd, ptr(nbr), ptr(inv_off), ptr(inv_ent), T, K, heads, dhp,
                                1.0 / math.sqrt(dh), ptr(g_ctx), hd, s3.ptr(), ptr(P), ptr(dS), ptr(work), ptr(g_qkv),
                                3 * hd, stream_ptr()), "wm3_bw_natten")
    cs, sn = _rope_pair_tables(extents, dh, dhp, dev)
    check(L.lib().wm3_bw_rope(ptr(g_qkv), 3 * hd, T, heads, dhp, ptr(cs), ptr(sn), stream_ptr()), "wm3_bw_rope")
    # ---- QKV ----
    s4 = _amax(g_qkv, T, 3 * hd)
    dwqkv = _gemm(_cast(g_qkv, T, 3 * hd, Tp, transpose=True, scale=s4), _cast(hn, T, kp, Tp, transpose=True),
                  3 * hd, kp, T)
    dbqkv = _colsum(g_qkv, T, 3 * hd)
    g_hn = _gemm(_cast(g_qkv, T, 3 * hd, 3 * hd, scale=s4), wt["w_qkv"], T, kp, 3 * hd)  # x s4
    # ---- LN1 (+ gx1) ----
    gx = torch.empty((T, D), dtype=torch.float32, device=dev)
    gxh1 = torch.empty_like(gx)
    gsc1 = torch.empty_like(gx)
    check(L.lib().wm3_bw_layernorm(ptr(xd), D, T, D, LN_EPS, ptr(bw.ln1_g), ptr(g_hn), kp, s4.ptr(), ptr(gx1),
                                   ptr(gx), ptr(gxh1), ptr(gsc1), stream_ptr()), "wm3_bw_layernorm")
    dln1_g = _colsum(gxh1, T, D)
    dln1_b = _colsum(gsc1, T, D)

    # ---- back to the reference layouts (float64, (in, out) matrices) ----
    def h(t, s=None):
        a = t.double().cpu().numpy()
        return a / s.value() if s is not None else a

    qk = _qk_perm(heads, dh, dhp)
    vv = _v_perm(heads, dh, dhp)
    Wqkv, Bqkv = h(dwqkv, s4)[:, :D], h(dbqkv)
    grads = {}
    for sec_i, (wn, bn, perm) in enumerate((("attn.wq", "attn.bq", qk), ("attn.wk", "attn.bk", qk),
                                            ("attn.wv", "attn.bv", vv))):
        rows = np.arange(hd) + sec_i * hd
        ok = perm >= 0
        gw = np.zeros((D, D))
        gb = np.zeros(D)
        gw[:, perm[ok]] = Wqkv[rows[ok]].T
        gb[perm[ok]] = Bqkv[rows[ok]]
        grads[wn], grads[bn] = gw, gb
    gwo = np.zeros((D, D))
    okv = vv >= 0
    gwo[vv[okv]] = h(dwo, s3)[:, okv].T
    grads["attn.wo"], grads["attn.bo"] = gwo, h(dbo)
    from .tensor import host_values
    hidden_mlp = host_values(params[f"{prefix}.mlp.w1"]).shape[1]
    grads["mlp.w1"] = h(dw1, s2)[:hidden_mlp, :D].T.copy()
    grads["mlp.b1"] = h(db1)[:hidden_mlp]
    grads["mlp.w2"] = h(dw2, s1)[:D, :hidden_mlp].T.copy()
    grads["mlp.b2"] = h(db2)
    grads["ln1.gain"], grads["ln1.bias"] = h(dln1_g), h(dln1_b)
    grads["ln2.gain"], grads["ln2.bias"] = h(dln2_g), h(dln2_b)
    names = dict(zip([n[len(prefix) + 1:] for n in block_param_names(prefix)], block_param_names(prefix)))
    return h(gx), {names[k]: np.ascontiguousarray(v) for k, v in grads.items()}
