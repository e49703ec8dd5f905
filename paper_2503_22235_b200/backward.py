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

    def inv(self) -> torch.Tensor:
        """1 / value() as a one-element device tensor (no host synchronisation)."""
        amax = self.bits.view(torch.float32)
        ok = (amax > 0) & torch.isfinite(amax)
        e = torch.where(ok, torch.ceil(torch.log2(torch.where(ok, amax, torch.ones_like(amax)))) - 14,
                        torch.zeros_like(amax))
        return torch.exp2(e)


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


def _colsum_amax(src: torch.Tensor, rows: int, cols: int, gelu_of: torch.Tensor | None = None,
                 bias: torch.Tensor | None = None, in_scale: _Scale | None = None):
    """(column sums, _Scale of max |v|) in one pass over v = src, or v = GELU backward of src (pre-activation
    `gelu_of` + bias, src divided by in_scale), which is then returned too: (colsum, scale, v)."""
    chunks = (rows + 255) // 256
    partial = torch.empty((chunks, cols), dtype=torch.float32, device=src.device)
    colsum = torch.empty(cols, dtype=torch.float32, device=src.device)
    s = _Scale(src.device)
    out = None if gelu_of is None else torch.empty((rows, cols), dtype=torch.float32, device=src.device)
    check(_lib.lib().wm3_bw_colsum_amax(ptr(src), src.stride(0), ptr(gelu_of),
                                        0 if gelu_of is None else gelu_of.stride(0), ptr(bias),
                                        None if in_scale is None else in_scale.ptr(), rows, cols, ptr(out),
                                        0 if out is None else out.stride(0), ptr(partial), ptr(colsum), s.ptr(),
                                        stream_ptr()), "wm3_bw_colsum_amax")
    return (colsum, s) if out is None else (colsum, s, out)


def _layernorm_backward(x: torch.Tensor, gamma: torch.Tensor, g: torch.Tensor, scale: _Scale,
                        add: torch.Tensor | None, gx_scale: _Scale | None = None):
    """LayerNorm reverse mode over rows of x [T][D] fp32 (autodiff.py:400-424) for the scaled output gradient g
    (row pitch g.stride(0)), plus `add` (the residual path): (gx, dgamma, dbeta), the parameter gradients as
    deterministic column sums of the kernel's per-row products.  (Folding those sums into the row kernel measured
    slower: a warp must then own a run of rows, which costs the occupancy the one-row-per-warp kernel hides its
    loads with.)  gx_scale (or None) receives max |gx| from the same kernel (the next cast's operand scale)."""
    T, D = x.shape
    dev = x.device
    gx = torch.empty((T, D), dtype=torch.float32, device=dev)
    gxh = torch.empty_like(gx)
    check(_lib.lib().wm3_bw_layernorm(ptr(x), x.stride(0), T, D, LN_EPS, ptr(gamma), ptr(g), g.stride(0),
                                      scale.ptr(), ptr(add), ptr(gx), ptr(gxh), None,
                                      None if gx_scale is None else gx_scale.ptr(), stream_ptr()),
          "wm3_bw_layernorm")
    # the bias gradient is the column sum of g / scale itself: no [T][D] copy of it
    return gx, _colsum(gxh, T, D), _colsum(g, T, D, scale=scale)


def _cast_colsum(src: torch.Tensor, rows: int, cols: int, ldd: int, scale: _Scale):
    """(16-bit operand copy of src[:rows, :cols] times the scale, zero padded to [rows][ldd]; column sums of src)
    in one pass — the producer already left max |src| in `scale`."""
    chunks = (rows + 255) // 256
    partial = torch.empty((chunks, cols), dtype=torch.float32, device=src.device)
    colsum = torch.empty(cols, dtype=torch.float32, device=src.device)
    out = torch.empty((rows, ldd), dtype=_lib.ELEM, device=src.device)
    check(_lib.lib().wm3_bw_cast_colsum(ptr(src), rows, cols, src.stride(0), ptr(out), ldd, scale.ptr(), ptr(partial),
                                        ptr(colsum), stream_ptr()), "wm3_bw_cast_colsum")
    return out, colsum


def _gemm_tn(a: torch.Tensor, b: torch.Tensor, m: int, n: int, k: int) -> torch.Tensor:
    """fp32 C[m][n] = sum_t A[t][:m] B[t][:n] over k rows (the weight gradients over tokens): MN-major tcgen05
    operands straight from the row-major 16-bit tensors, no transposed copies; the token range split over the CTA
    pairs when the weight has few output tiles (deterministic ordered sum of the partials)."""
    out = torch.empty((m, n), dtype=torch.float32, device=a.device)
    sp = _lib.lib().wm3_linear_tn_split_count(m, n, k)  # split-K partial planes the library will use
    scratch = torch.empty(sp * m * n, dtype=torch.float32, device=a.device) if sp > 1 else None
    check(_lib.lib().wm3_linear_tn_split(ptr(a), a.stride(0), ptr(b), b.stride(0), m, n, k, ptr(out), out.stride(0),
                                         ptr(scratch), 0 if scratch is None else scratch.numel(), stream_ptr()),
          "wm3_linear_tn_split")
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


_ROPE_PAIRS: dict = {}


class _TcAttention:
    """Per-geometry state of the tensor-core attention backward (wm3_natten_bwd): the CSR of chunk slots per key
    token (fixed order: the deterministic dK / dV reduction), the partial scratch and the small operand buffers.
    None when the geometry is unsupported (head dim padded to 64, or the window mask does not fit the MMA bias
    step) or WM3_BW_NA=cuda selects the CUDA-core kernels (A/B aid)."""

    _cache: dict = {}

    @classmethod
    def get(cls, extents, window, heads: int, dhp: int):
        import os
        if os.environ.get("WM3_BW_NA", "tc") == "cuda":
            return None
        key = (tuple(extents), tuple(window), heads, dhp, torch.cuda.current_device())
        if key not in cls._cache:
            cls._cache[key] = cls._build(extents, window, heads, dhp)
        return cls._cache[key]

    @classmethod
    def _build(cls, extents, window, heads: int, dhp: int):
        import ctypes
        d, h, w = (int(e) for e in extents)
        wd, wh, ww = (int(e) for e in window)
        nt, mc, sup = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(_lib.lib().wm3_natten_bwd_info(d, h, w, heads, dhp, wd, wh, ww, ctypes.byref(nt), ctypes.byref(mc),
                                             ctypes.byref(sup), stream_ptr()), "wm3_natten_bwd_info")
        if not sup.value:
            return None
        ntiles, maxch = nt.value, mc.value
        table = torch.empty(ntiles * maxch * 128, dtype=torch.int32, device="cuda")
        check(_lib.lib().wm3_natten_slot_table(d, h, w, heads, dhp, wd, wh, ww, ptr(table), stream_ptr()),
              "wm3_natten_slot_table")
        tab = table.cpu().numpy()
        t_count = d * h * w
        codes = np.nonzero(tab >= 0)[0]
        toks = tab[codes]
        order = np.argsort(toks, kind="stable")  # by key token, then (tile, chunk, slot)
        off = np.zeros(t_count + 1, dtype=np.int32)
        np.cumsum(np.bincount(toks, minlength=t_count), out=off[1:])
        st = cls()
        st.ntiles, st.maxch = ntiles, maxch
        st.off = torch.from_numpy(off).cuda()
        st.ent = torch.from_numpy(codes[order].astype(np.int32)).cuda()
        st.partial = torch.empty(ntiles * heads * maxch * 2 * 2 * 64 * dhp, dtype=torch.float32, device="cuda")
        st.maxima = torch.zeros(2, dtype=torch.int32, device="cuda")
        st.factors = torch.zeros(2, dtype=torch.float32, device="cuda")
        return st


def _rope_pair_tables(extents, dh: int, dhp: int, dev) -> tuple[torch.Tensor, torch.Tensor]:
    """cos / sin (T, dhp / 2) of the interleaved pairs (pair j = reference columns (j, j + dh/2), attention.py:48-92);
    padding pairs are the identity.  Built once per geometry and device."""
    key = (tuple(extents), dh, dhp, str(dev))
    hit = _ROPE_PAIRS.get(key)
    if hit is None:
        hit = _ROPE_PAIRS[key] = _rope_pair_tables_build(extents, dh, dhp, dev)
    return hit


def _rope_pair_tables_build(extents, dh: int, dhp: int, dev) -> tuple[torch.Tensor, torch.Tensor]:
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


class BlockGrads:
    """Device fp32 accumulators of one block's parameter gradients, in the kernel layouts (padded, q/k pairs
    interleaved) and unscaled; `add` sums repeated applications of the block (a rollout reuses its processor)."""

    def __init__(self):
        self.t: dict = {}

    def add(self, name: str, g: torch.Tensor, scale: _Scale | None = None) -> None:
        if scale is not None:
            g = g * scale.inv()
        cur = self.t.get(name)
        if cur is None:
            self.t[name] = g.clone() if scale is None else g
        else:
            cur.add_(g)


def block_vjp_device(xd: torch.Tensor, bw, extents, window, heads: int, dh: int, gyd: torch.Tensor,
                     acc: BlockGrads) -> torch.Tensor:
    """Device reverse mode of one block: returns gx (fp32, (T, hidden)) for the output cotangent gyd and adds the
    parameter gradients to `acc`.  Forward recompute from the block input xd (nothing else is saved, like a
    checkpointed segment, autodiff.py:893-924); one stream, no host synchronisation."""
    T, D = xd.shape
    dev = xd.device
    dhp, hd, kp, np_, nm = bw.dhp, bw.heads * bw.dhp, bw.kp, bw.np_, bw.nm
    L = _lib
    wt = _transposed_weights(bw)
    rope = CACHE.rope(extents, dh)
    # ---- forward recompute (the kernels of the block forward, keeping the intermediates) ----
    hn = ops.layernorm_bf16(xd, bw.ln1_g, bw.ln1_b, ldo=kp)
    grid = ops.KVGrid(extents, window)
    qkv = torch.zeros((grid.tokens, 3 * hd), dtype=L.ELEM, device=dev)
    ops.linear_grid(hn, bw.w_qkv, L.WM3_EPI_QKV_ROPE, bw.b_qkv, qkv, grid, rope=rope.struct(extents, 0, heads, dhp))
    tca = _TcAttention.get(extents, window, heads, dhp)
    if tca is not None:
        ctx = torch.empty((T, hd), dtype=L.ELEM, device=dev)
        lse = torch.empty((T, heads), dtype=torch.float32, device=dev)
        check(L.lib().wm3_natten_fwd_lse(ptr(qkv), qkv.stride(0), ptr(ctx), ctx.stride(0), *extents, heads, dhp,
                                         *window, 1.0 / math.sqrt(dh), ptr(lse), stream_ptr()), "wm3_natten_fwd_lse")
    else:
        ctx = ops.natten(qkv, grid, heads, dhp, dh, window)
    x1 = xd.clone()
    ops.linear(ctx, bw.w_o, L.WM3_EPI_BIAS_RESID_F32, bias=bw.b_o, out=x1, n_valid=D)
    hn2 = ops.layernorm_bf16(x1, bw.ln2_g, bw.ln2_b, ldo=kp)
    a0 = _gemm(hn2, bw.w_1, T, nm, kp)                                   # W1 pre-activation without bias
    mid = torch.empty((T, nm), dtype=L.ELEM, device=dev)                # GELU output as the forward stores it
    check(L.lib().wm3_bw_gelu_fwd(ptr(a0), nm, ptr(bw.b_1), T, nm, ptr(mid), nm, stream_ptr()), "wm3_bw_gelu_fwd")

    # ---- W2 ----
    db2, s1 = _colsum_amax(gyd, T, D)
    gyh = _cast(gyd, T, D, kp, scale=s1)                                # zero-padded to kp >= np_
    dw2 = _gemm_tn(gyh, mid, kp, nm, T)                                 # (kp, nm), x s1
    # ---- GELU' and W1 ----
    # g_a = (gy . W2) / s1 * gelu'(a0 + b1), the GELU backward in the gradient GEMM's epilogue, in place over a0
    # (and its max |.| for the operand scale s2: every gradient's scale comes from its producer, so the cast and
    # the bias gradient are one pass over it)
    s2 = _Scale(dev)
    check(L.lib().wm3_linear_gelu_grad(ptr(gyh), gyh.stride(0), ptr(wt["w_2"]), wt["w_2"].stride(0), T, nm, np_,
                                       ptr(a0), a0.stride(0), ptr(bw.b_1), s1.ptr(), s2.ptr(), stream_ptr()),
          "wm3_linear_gelu_grad")
    g_a, a0 = a0, None
    gah, db1 = _cast_colsum(g_a, T, nm, nm, s2)
    dw1 = _gemm_tn(gah, hn2, nm, kp, T)
    g_hn2 = _gemm(gah, wt["w_1"], T, kp, nm)   # x s2
    # ---- LN2 (+ the residual path gy) ----
    s3 = _Scale(dev)
    gx1, dln2_g, dln2_b = _layernorm_backward(x1, bw.ln2_g, g_hn2, s2, gyd, gx_scale=s3)
    # ---- O-proj ----
    gx1h, dbo = _cast_colsum(gx1, T, D, kp, s3)
    dwo = _gemm_tn(gx1h, ctx, kp, hd, T)
    g_ctx = _gemm(gx1h, wt["w_o"], T, hd, np_)  # x s3
    # ---- attention (query and key sides) and the rotary transpose ----
    cs, sn = _rope_pair_tables(extents, dh, dhp, dev)
    s4 = _Scale(dev)  # max |g_qkv|, left by the kernels that write it (tensor-core path)
    if tca is not None:
        g_qkv = torch.empty((T, 3 * hd), dtype=torch.float32, device=dev)  # every element written below
        # tensor cores: dQ per query tile, dK / dV as deterministic sums of per-chunk partials (natten.cu)
        dout = torch.empty((T, hd), dtype=L.ELEM, device=dev)
        check(L.lib().wm3_bw_na_prep(ptr(qkv), 3 * hd, T, heads, dhp, ptr(g_ctx), hd, s3.ptr(), 1.0 / math.sqrt(dh),
                                     ptr(dout), hd, ptr(tca.maxima), ptr(tca.factors), stream_ptr()), "wm3_bw_na_prep")
        check(L.lib().wm3_natten_bwd(ptr(qkv), 3 * hd, ptr(dout), hd, ptr(ctx), hd, ptr(lse), ptr(g_qkv), 3 * hd,
                                     ptr(tca.partial), ptr(tca.off), ptr(tca.ent), ptr(tca.factors), ptr(cs), ptr(sn),
                                     s4.ptr(), *extents, heads, dhp, *window, 1.0 / math.sqrt(dh), stream_ptr()),
              "wm3_natten_bwd")  # dK leaves through the rotary transpose (coalesced per key in the reduction)
        check(L.lib().wm3_bw_rope_q(ptr(g_qkv), 3 * hd, T, heads, dhp, ptr(cs), ptr(sn), s4.ptr(), stream_ptr()),
              "wm3_bw_rope_q")
    else:
        g_qkv = torch.zeros((T, 3 * hd), dtype=torch.float32, device=dev)
        nbr, inv_off, inv_ent, K = _InverseNeighbors.get(extents, window)
        P = torch.empty((T, heads, K), dtype=torch.float32, device=dev)
        dS = torch.empty_like(P)
        work = torch.empty((T, heads, 2 * K), dtype=torch.float32, device=dev)
        check(L.lib().wm3_bw_natten(ptr(qkv), 3 * hd, ptr(nbr), ptr(inv_off), ptr(inv_ent), T, K, heads, dhp,
                                    1.0 / math.sqrt(dh), ptr(g_ctx), hd, s3.ptr(), ptr(P), ptr(dS), ptr(work),
                                    ptr(g_qkv), 3 * hd, stream_ptr()), "wm3_bw_natten")
        check(L.lib().wm3_bw_rope(ptr(g_qkv), 3 * hd, T, heads, dhp, ptr(cs), ptr(sn), stream_ptr()), "wm3_bw_rope")
        check(L.lib().wm3_bw_amax(ptr(g_qkv), T, 3 * hd, g_qkv.stride(0), s4.ptr(), stream_ptr()), "wm3_bw_amax")
    # ---- QKV ----
    gqh, dbqkv = _cast_colsum(g_qkv, T, 3 * hd, 3 * hd, s4)
    dwqkv = _gemm_tn(gqh, hn, 3 * hd, kp, T)
    g_hn = _gemm(gqh, wt["w_qkv"], T, kp, 3 * hd)  # x s4
    # ---- LN1 (+ gx1) ----
    gx, dln1_g, dln1_b = _layernorm_backward(xd, bw.ln1_g, g_hn, s4, gx1)

    acc.add("w_qkv", dwqkv, s4)
    acc.add("b_qkv", dbqkv)
    acc.add("w_o", dwo, s3)
    acc.add("b_o", dbo)
    acc.add("w_1", dw1, s2)
    acc.add("b_1", db1)
    acc.add("w_2", dw2, s1)
    acc.add("b_2", db2)
    acc.add("ln1_g", dln1_g)
    acc.add("ln1_b", dln1_b)
    acc.add("ln2_g", dln2_g)
    acc.add("ln2_b", dln2_b)
    return gx


def block_grads_to_reference(acc: BlockGrads, bw, params: dict, prefix: str, dh: int, hidden: int) -> dict:
    """The accumulated kernel-layout gradients in the reference's layouts: float64, (in, out) matrices, parameter
    names of attention.py:105-139.  The re-layout (q / k pair de-interleaving, head padding, transposes) runs on the
    device in fp32 (exact copies); one page-locked download per tensor, float64 on the host."""
    D = hidden
    heads, dhp = bw.heads, bw.dhp
    hd = heads * dhp
    g = acc.t
    dev = g["w_qkv"].device
    from .tensor import host_values
    hidden_mlp = host_values(params[f"{prefix}.mlp.w1"]).shape[1]
    qk = _qk_perm(heads, dh, dhp)
    vv = _v_perm(heads, dh, dhp)
    out: dict = {}
    for sec_i, (wn, bn, perm) in enumerate((("attn.wq", "attn.bq", qk), ("attn.wk", "attn.bk", qk),
                                            ("attn.wv", "attn.bv", vv))):
        ok = np.nonzero(perm >= 0)[0]
        src = torch.from_numpy(ok + sec_i * hd).to(dev)
        dst = torch.from_numpy(perm[ok]).to(dev)
        gw = torch.zeros((D, D), dtype=torch.float32, device=dev)
        gb = torch.zeros(D, dtype=torch.float32, device=dev)
        gw[:, dst] = g["w_qkv"][src, :D].t()
        gb[dst] = g["b_qkv"][src]
        out[wn], out[bn] = gw, gb
    okv = np.nonzero(vv >= 0)[0]
    gwo = torch.zeros((D, D), dtype=torch.float32, device=dev)
    gwo[torch.from_numpy(vv[okv]).to(dev)] = g["w_o"][:D, torch.from_numpy(okv).to(dev)].t()
    out["attn.wo"], out["attn.bo"] = gwo, g["b_o"][:D]
    out["mlp.w1"] = g["w_1"][:hidden_mlp, :D].t()
    out["mlp.b1"] = g["b_1"][:hidden_mlp]
    out["mlp.w2"] = g["w_2"][:D, :hidden_mlp].t()
    out["mlp.b2"] = g["b_2"][:D]
    out["ln1.gain"], out["ln1.bias"] = g["ln1_g"][:D], g["ln1_b"][:D]
    out["ln2.gain"], out["ln2.bias"] = g["ln2_g"][:D], g["ln2_b"][:D]
    names = dict(zip([n[len(prefix) + 1:] for n in block_param_names(prefix)], block_param_names(prefix)))
    # one float64 buffer on the device (exact widening) and one download into page-locked host memory (torch's
    # caching host allocator hands the same blocks back call after call); the returned arrays are views of it
    keys = list(out)
    flat = torch.cat([out[k].reshape(-1) for k in keys]).to(torch.float64)
    hv = _to_host_f64(flat)
    res, o = {}, 0
    for k in keys:
        n = out[k].numel()
        res[names[k]] = hv[o:o + n].reshape(tuple(out[k].shape))
        o += n
    return res


def _to_host_f64(t: torch.Tensor) -> np.ndarray:
    """float64 numpy copy through page-locked memory (tensor.device_to_host_f64)."""
    from .tensor import device_to_host_f64
    return device_to_host_f64(t)


def block_vjp(x, params: dict, prefix: str, extents, window, heads: int, gy):
    """(gx, grads) of y = natten_block(x) for the output gradient gy; numpy float64 in the reference layouts."""
    from .attention import to_device_f32, validate_block_args
    extents = tuple(int(e) for e in extents)
    window = tuple(int(w) for w in window)
    xd = to_device_f32(x)
    dh = validate_block_args(tuple(xd.shape), extents, window, heads)
    bw = CACHE.block(params, prefix, heads)
    acc = BlockGrads()
    gx = block_vjp_device(xd, bw, extents, window, heads, dh, to_device_f32(gy), acc)
    return _to_host_f64(gx), block_grads_to_reference(acc, bw, params, prefix, dh, xd.shape[1])


# ------------------------------------------------------------------------------------------------------------
# Reverse mode of the latent rollout with checkpointed blocks and host offload
# ------------------------------------------------------------------------------------------------------------
class DeviceActivationStore:
    """Saved block inputs kept in HBM: plain per-block checkpointing (autodiff.py:893-924), one latent per block."""

    def __init__(self):
        self.slots: dict = {}
        self.resident = 0
        self.high_water = 0
        self.demand_stalls = 0

    def put(self, k: int, x: torch.Tensor) -> None:
        self.slots[k] = x.clone()
        self.resident += x.numel() * x.element_size()
        self.high_water = max(self.high_water, self.resident)

    def begin_backward(self, order) -> None:
        pass

    def take(self, k: int) -> torch.Tensor:
        return self.slots[k]

    def release(self, k: int) -> None:
        x = self.slots.pop(k)
        self.resident -= x.numel() * x.element_size()

    def stats(self) -> dict:
        return {"kind": "device", "high_water_bytes": self.high_water, "demand_stalls": 0}


class HostOffloadStore:
    """Saved block inputs in page-locked host memory, moved on a side CUDA stream: the B200 counterpart of the
    reference's OffloadEngine / PrefetchPipeline (offload.py:287-412, 226-285).

    Forward, put(k, x): x is staged into one of `lookahead + 1` device ring slots on the compute stream (the slot
    is reused only after its previous device-to-host copy completed), and the side stream copies the slot out to
    the host.  Backward, in the order given to begin_backward(): the side stream brings inputs back into the ring
    `lookahead` blocks ahead of need (each slot reused once the compute stream's recompute of its previous block
    is done), take(k) makes the compute stream wait for that copy, release(k) frees the slot and issues the next
    prefetch.  Transfers overlap recompute; device residency of saved inputs is the ring, whatever the number of
    blocks; the bytes are exact copies, so gradients are bitwise those of the in-HBM store."""

    def __init__(self, shape, lookahead: int = 2):
        if lookahead < 1:
            raise ValueError(f"lookahead must be >= 1, got {lookahead}")
        self.shape = tuple(shape)
        self.lookahead = int(lookahead)
        self.side = torch.cuda.Stream()
        self.ring = [torch.empty(self.shape, dtype=torch.float32, device="cuda") for _ in range(self.lookahead + 1)]
        self.slot_free = [None] * len(self.ring)  # event after the last use of the slot (any stream)
        self.host: dict = {}
        self.ready: dict = {}  # k -> (slot, event) of a fetched input
        self.order: list = []
        self.next_fetch = 0
        self.demand_stalls = 0
        self.transfers = 0
        self.high_water = len(self.ring) * self.ring[0].numel() * 4

    def _wait_slot(self, stream, i: int) -> None:
        if self.slot_free[i] is not None:
            stream.wait_event(self.slot_free[i])

    def put(self, k: int, x: torch.Tensor) -> None:
        i = k % len(self.ring)
        main = torch.cuda.current_stream()
        self._wait_slot(main, i)
        self.ring[i].copy_(x)
        staged = torch.cuda.Event()
        staged.record(main)
        h = self.host.get(k)
        if h is None:
            h = torch.empty(self.shape, dtype=torch.float32, pin_memory=True)
            self.host[k] = h
        with torch.cuda.stream(self.side):
            self.side.wait_event(staged)
            h.copy_(self.ring[i], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.side)
        self.slot_free[i] = done
        self.transfers += 1

    def begin_backward(self, order) -> None:
        self.order = list(order)
        self.next_fetch = 0
        self.occupied: set = set()  # ring slots holding a fetched input not yet released
        for _ in range(min(self.lookahead, len(self.order))):
            self._prefetch()

    def _slot(self, grow: bool):
        """A ring slot no fetched-but-unreleased input holds; with grow, a new slot when all are taken (an
        out-of-order request beyond the lookahead), else None."""
        for i in range(len(self.ring)):
            if i not in self.occupied:
                return i
        if not grow:
            return None
        self.ring.append(torch.empty(self.shape, dtype=torch.float32, device="cuda"))
        self.slot_free.append(None)
        self.high_water = max(self.high_water, len(self.ring) * self.ring[0].numel() * 4)
        return len(self.ring) - 1

    def _fetch(self, k: int, i: int) -> None:
        with torch.cuda.stream(self.side):
            self._wait_slot(self.side, i)
            self.ring[i].copy_(self.host[k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.side)
        self.ready[k] = (i, ev)
        self.occupied.add(i)
        self.transfers += 1

    def _prefetch(self) -> None:
        while self.next_fetch < len(self.order) and self.order[self.next_fetch] in self.ready:
            self.next_fetch += 1
        if self.next_fetch >= len(self.order):
            return
        i = self._slot(grow=False)
        if i is None:
            return
        k = self.order[self.next_fetch]
        self.next_fetch += 1
        self._fetch(k, i)

    def take(self, k: int) -> torch.Tensor:
        if k not in self.ready:  # not prefetched (out-of-order request): fetch on demand
            self.demand_stalls += 1
            self._fetch(k, self._slot(grow=True))
        i, ev = self.ready[k]
        torch.cuda.current_stream().wait_event(ev)
        return self.ring[i]

    def release(self, k: int) -> None:
        i, _ = self.ready.pop(k)
        self.occupied.discard(i)
        done = torch.cuda.Event()
        done.record(torch.cuda.current_stream())
        self.slot_free[i] = done
        self._prefetch()

    def stats(self) -> dict:
        return {"kind": "host", "high_water_bytes": self.high_water, "demand_stalls": self.demand_stalls,
                "transfers": self.transfers, "lookahead": self.lookahead}


def rollout_vjp(z0, plan, params: dict, cfg, g_out, offload: bool = False, lookahead: int = 2,
                reference_grads: bool = True):
    """Reverse mode of the greedy latent rollout (rollout.py:56-81) on the device.

    z0: the initial latent tokens (T, hidden); plan: processor horizons in order (e.g. (6, 6, 1)); g_out: the
    cotangent of the final latent tokens.  Returns (z_final, dL/dz0, {parameter name: gradient}, store stats):
    z_final as a device fp32 tensor, dL/dz0 as float64 numpy, every processor block's parameter gradients summed
    over the steps that applied it (float64, the reference's layouts).  Like the reference's checkpoint_segment
    per block (autodiff.py:893-924) the forward keeps only each block's input and the backward recomputes the
    block from it (block_vjp_device); with offload=True those inputs live in page-locked host memory and return
    `lookahead` blocks ahead of need (HostOffloadStore), bitwise the same gradients as offload=False.
    reference_grads=False returns the device accumulators ({block prefix: BlockGrads}, kernel layouts) and dL/dz0
    as a device tensor instead, for a training loop that stays on the device.
    """
    from .attention import to_device_f32
    from .blocks import block_forward
    from .config import as_config
    cfg = as_config(cfg)
    ext, win, heads, dh = cfg.latent_extents, cfg.window, cfg.heads, cfg.head_dim
    for h in plan:
        if f"proc{h}.blk0.ln1.gain" not in params:
            from .errors import ConfigError
            raise ConfigError(f"parameters carry no {h} h processor")
    prefixes = [f"proc{h}.blk{i}" for h in plan for i in range(cfg.proc_blocks)]
    x = to_device_f32(z0)
    store = HostOffloadStore(x.shape, lookahead) if offload else DeviceActivationStore()
    rope = CACHE.rope(ext, dh)
    for k, pre in enumerate(prefixes):
        bw = CACHE.block(params, pre, heads)
        store.put(k, x)
        block_forward(x, bw, CACHE.workspace(ext, win, bw), rope, ext, win)
    z = x
    g = to_device_f32(g_out)
    accs: dict = {}
    order = list(reversed(range(len(prefixes))))
    store.begin_backward(order)
    for k in order:
        pre = prefixes[k]
        bw = CACHE.block(params, pre, heads)
        xk = store.take(k)
        g = block_vjp_device(xk, bw, ext, win, heads, dh, g, accs.setdefault(pre, BlockGrads()))
        store.release(k)
    if not reference_grads:
        return z, g, accs, store.stats()
    grads: dict = {}
    for pre, acc in accs.items():
        grads.update(block_grads_to_reference(acc, CACHE.block(params, pre, heads), params, pre, dh, cfg.hidden))
    torch.cuda.synchronize()
    return z, _to_host_f64(g), grads, store.stats()
