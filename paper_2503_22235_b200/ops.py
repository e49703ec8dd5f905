"""Device-level operator wrappers over libwm3.so (torch tensors in/out, all on the current stream).

Torch is only the allocator and stream provider here; every op below is one launch of a hand-written
sm_100a kernel from csrc/.  Shapes are validated before launch; kernel faults raise RuntimeError.
"""

from __future__ import annotations

import math

import torch

from . import _lib
from ._lib import check, ptr, stream_ptr


def _req(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if not t.is_cuda:
        raise RuntimeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise RuntimeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise RuntimeError(f"{name} must be a row-major 2D tensor")


def neighbor_table(extents, window, row0: int = 0, nrows: int | None = None) -> torch.Tensor:
    """(T, K) int64 neighbor table computed on the GPU (grid.py:107-130 semantics)."""
    d, h, w = (int(e) for e in extents)
    wd, wh, ww = (int(e) for e in window)
    nrows = h if nrows is None else int(nrows)
    out = torch.empty((d * nrows * w, wd * wh * ww), dtype=torch.int64, device="cuda")
    check(_lib.lib().wm3_neighbor_table(d, h, w, wd, wh, ww, int(row0), nrows, ptr(out), stream_ptr()),
          "wm3_neighbor_table")
    return out


def natten_windows(extents, window, rows_global: int | None = None, row0: int = 0) -> torch.Tensor:
    d, h, w = (int(e) for e in extents)
    wd, wh, ww = (int(e) for e in window)
    rg = h if rows_global is None else int(rows_global)
    out = torch.empty((d * h * w, 3), dtype=torch.int32, device="cuda")
    check(_lib.lib().wm3_natten_windows(d, h, w, rg, int(row0), wd, wh, ww, ptr(out), stream_ptr()),
          "wm3_natten_windows")
    return out


def layernorm_bf16(x: torch.Tensor, gain: torch.Tensor, bias: torch.Tensor, ldo: int | None = None,
                   out: torch.Tensor | None = None, eps: float = 1e-6) -> torch.Tensor:
    _req(x, torch.float32, "x")
    m, n = x.shape
    ldo = n if ldo is None else int(ldo)
    if out is None:
        out = torch.empty((m, ldo), dtype=_lib.ELEM, device=x.device)
    check(_lib.lib().wm3_layernorm_bf16(ptr(x), x.stride(0), m, n, ptr(gain), ptr(bias), float(eps), ptr(out),
                                        out.stride(0), stream_ptr()), "wm3_layernorm_bf16")
    return out


def ln_fold_consumer(row_stats: torch.Tensor, fold_c: torch.Tensor) -> "_lib.LnFoldT":
    """wm3_ln_fold_t for a GEMM that applies the folded LayerNorm (reads (rstd, rstd * mean) per row)."""
    _req(row_stats, torch.float32, "row_stats")
    return _lib.LnFoldT(None, 0, None, row_stats.data_ptr(), fold_c.data_ptr())


def ln_fold_producer(xh: torch.Tensor, stats: torch.Tensor) -> "_lib.LnFoldT":
    """wm3_ln_fold_t for a residual GEMM that also writes the fp16 copy of x and its row statistics."""
    _req(xh, _lib.ELEM, "xh")
    _req(stats, torch.float32, "stats")
    return _lib.LnFoldT(xh.data_ptr(), xh.stride(0), stats.data_ptr(), None, None)


def ln_fold_prep(x: torch.Tensor, n: int, xh: torch.Tensor, row_stats: torch.Tensor, eps: float = 1e-6) -> None:
    """Start of a folded chain: xh = fp16(x) (pad columns zero) and x's (rstd, rstd * mean) per row."""
    _req(x, torch.float32, "x")
    _req(xh, _lib.ELEM, "xh")
    check(_lib.lib().wm3_ln_fold_prep(ptr(x), x.stride(0), x.shape[0], int(n), ptr(xh), xh.stride(0), float(eps),
                                      ptr(row_stats), stream_ptr()), "wm3_ln_fold_prep")


def ln_fold_finalize(stats: torch.Tensor, parts: int, n: int, row_stats: torch.Tensor, eps: float = 1e-6) -> None:
    """Producer partial sums -> (rstd, rstd * mean) per row."""
    check(_lib.lib().wm3_ln_fold_finalize(ptr(stats), int(parts), int(n), float(eps), stats.shape[0],
                                          ptr(row_stats), stream_ptr()), "wm3_ln_fold_finalize")


def linear(a: torch.Tensor, w: torch.Tensor, epi: int, bias: torch.Tensor | None = None,
           out: torch.Tensor | None = None, n_valid: int | None = None,
           rope: "_lib.RopeT | None" = None, fold: "_lib.LnFoldT | None" = None) -> torch.Tensor:
    """out = epilogue(a @ w.T + bias); a (M, K) bf16, w (N, K) bf16 (weights stored (out, in)).  fold: the
    folded-LayerNorm producer / consumer descriptor (ln_fold_producer / ln_fold_consumer)."""
    _req(a, _lib.ELEM, "a")
    _req(w, _lib.ELEM, "w")
    m, k = a.shape
    n, k2 = w.shape
    if k2 != k:
        raise RuntimeError(f"linear: inner extents differ {a.shape} @ {w.shape}^T")
    f32_out = epi in (_lib.WM3_EPI_F32, _lib.WM3_EPI_BIAS_RESID_F32)
    if out is None:
        if epi == _lib.WM3_EPI_BIAS_RESID_F32:
            raise RuntimeError("residual epilogue needs the fp32 stream as `out`")
        out = torch.empty((m, n), dtype=torch.float32 if f32_out else _lib.ELEM, device=a.device)
    _req(out, torch.float32 if f32_out else _lib.ELEM, "out")
    nv = out.shape[1] if n_valid is None else int(n_valid)
    rp = None if rope is None else ctypes_byref(rope)
    if fold is not None:
        check(_lib.lib().wm3_linear_fold(ptr(a), a.stride(0), ptr(w), w.stride(0), m, n, k, int(epi), ptr(out),
                                         out.stride(0), nv, ptr(bias), rp, 1, m, m, 0, None, ctypes_byref(fold),
                                         stream_ptr()), "wm3_linear_fold")
        return out
    check(_lib.lib().wm3_linear(ptr(a), a.stride(0), ptr(w), w.stride(0), m, n, k, int(epi), ptr(out),
                                out.stride(0), nv, ptr(bias), rp, stream_ptr()), "wm3_linear")
    return out


def ctypes_byref(obj):
    import ctypes
    return ctypes.byref(obj)


class KVGrid:
    """Geometry of the K/V token grid consumed by the fused attention kernel.

    Tokens live at [depth][halo_lo + rows + halo_hi][cols]: the band's own rows plus latitude-band halo rows
    received from the neighbouring bands (none on a single GPU).  Longitude wrap needs no padding: the
    kernel fetches a seam-crossing key patch as two TMA boxes.  `batch` latents (ensemble members) are
    stacked member-major along depth: member b owns planes [b * depth, (b + 1) * depth).
    """

    def __init__(self, extents, window=None, halo_lo: int = 0, halo_hi: int = 0, batch: int = 1):
        self.depth, self.rows, self.cols = (int(e) for e in extents)
        self.halo_lo, self.halo_hi = int(halo_lo), int(halo_hi)
        self.batch = int(batch)
        self.rows_ext = self.rows + self.halo_lo + self.halo_hi

    @property
    def planes(self) -> int:
        return self.batch * self.depth

    @property
    def tokens(self) -> int:
        return self.planes * self.rows_ext * self.cols

    def interior(self, buf: torch.Tensor) -> torch.Tensor:
        """(batch * T, C) copy of the band's own tokens in token order (debug / probes)."""
        g = buf.view(self.planes, self.rows_ext, self.cols, -1)
        return g[:, self.halo_lo:self.halo_lo + self.rows].reshape(self.planes * self.rows * self.cols, -1)


def linear_grid(a: torch.Tensor, w: torch.Tensor, epi: int, bias: torch.Tensor, out: torch.Tensor, grid: KVGrid,
                rope: "_lib.RopeT | None" = None, halo: "_lib.HaloT | None" = None,
                fold: "_lib.LnFoldT | None" = None) -> torch.Tensor:
    """linear() whose output rows (band tokens) land in the K/V grid `out` (halo rows left untouched).  With
    `halo` (wm3_halo_t), the QKV epilogue also stores the band's boundary K/V rows into the neighbouring bands'
    grids (fused halo exchange over peer memory)."""
    _req(a, _lib.ELEM, "a")
    _req(w, _lib.ELEM, "w")
    _req(out, _lib.ELEM, "out")
    m, k = a.shape
    n = w.shape[0]
    rp = None if rope is None else ctypes_byref(rope)
    plane = grid.rows * grid.cols
    args = (ptr(a), a.stride(0), ptr(w), w.stride(0), m, n, k, int(epi), ptr(out), out.stride(0), out.shape[1],
            ptr(bias), rp, grid.planes, plane, grid.rows_ext * grid.cols, grid.halo_lo * grid.cols)
    if fold is not None:
        check(_lib.lib().wm3_linear_fold(*args, None if halo is None else ctypes_byref(halo), ctypes_byref(fold),
                                         stream_ptr()), "wm3_linear_fold")
    elif halo is None:
        check(_lib.lib().wm3_linear_planes(*args, stream_ptr()), "wm3_linear_planes")
    else:
        check(_lib.lib().wm3_linear_planes_halo(*args, ctypes_byref(halo), stream_ptr()), "wm3_linear_planes_halo")
    return out


def natten(qkv: torch.Tensor, grid: KVGrid, heads: int, dhp: int, dh: int, window,
           out: torch.Tensor | None = None, rows_global: int | None = None, row0: int = 0,
           q_rows: tuple[int, int] | None = None) -> torch.Tensor:
    """Fused neighborhood attention over the padded qkv grid -> ctx (T, heads*dhp) bf16, band token order.
    q_rows = (lo, hi): only the queries of global rows [lo, hi) (wm3_natten_fwd_rows; other rows untouched)."""
    _req(qkv, _lib.ELEM, "qkv")
    if qkv.shape[0] != grid.tokens:
        raise RuntimeError(f"qkv has {qkv.shape[0]} rows, padded grid needs {grid.tokens}")
    wd, wh, ww = (int(e) for e in window)
    d, h, w = grid.depth, grid.rows, grid.cols
    rg = h if rows_global is None else int(rows_global)
    t = grid.batch * d * h * w
    if out is None:
        out = torch.empty((t, heads * dhp), dtype=_lib.ELEM, device=qkv.device)
    _req(out, _lib.ELEM, "out")
    if q_rows is not None:
        lo, hi = int(q_rows[0]), int(q_rows[1])
        check(_lib.lib().wm3_natten_fwd_rows(ptr(qkv), qkv.stride(0), ptr(out), out.stride(0), grid.batch, d, h, w, rg,
                                             int(row0), grid.halo_lo, grid.halo_hi, int(heads), int(dhp), wd, wh, ww,
                                             float(1.0 / math.sqrt(dh)), lo, hi - lo, stream_ptr()),
              "wm3_natten_fwd_rows")
        return out
    check(_lib.lib().wm3_natten_fwd(ptr(qkv), qkv.stride(0), ptr(out), out.stride(0), grid.batch, d, h, w, rg,
                                    int(row0),
                                    grid.halo_lo, grid.halo_hi, int(heads), int(dhp), wd, wh, ww,
                                    float(1.0 / math.sqrt(dh)), stream_ptr()), "wm3_natten_fwd")
    return out


def pad_tokens_to_grid(x: torch.Tensor, grid: KVGrid) -> torch.Tensor:
    """Place token-ordered rows (T, C) into a fresh K/V grid buffer (tests)."""
    buf = torch.zeros((grid.tokens, x.shape[1]), dtype=x.dtype, device=x.device)
    g = buf.view(grid.depth, grid.rows_ext, grid.cols, -1)
    g[:, grid.halo_lo:grid.halo_lo + grid.rows] = x.view(grid.depth, grid.rows, grid.cols, -1)
    return buf
