"""ctypes binding of libwm3.so, the C ABI declared in include/wm3.h.

There is no fallback: if the shared library is missing or CUDA is unavailable, every entry point
raises.  Status codes from the library become RuntimeError carrying wm3_last_error().
"""

from __future__ import annotations

import ctypes
import os
from functools import lru_cache

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WM3_LIB") or os.path.join(_HERE, "libwm3.so")  # WM3_LIB: A/B builds (profiling)

# Tensor-core operand dtype the library is built for (csrc/common.cuh elem_t): fp16 by default.  load_library()
# checks it against the library's own wm3_operand_dtype() and refuses a mismatched build.
ELEM = torch.float16
WM3_DTYPE_F16, WM3_DTYPE_BF16 = 1, 2

WM3_EPI_F32 = 0
WM3_EPI_BIAS_BF16 = 1
WM3_EPI_BIAS_GELU_BF16 = 2
WM3_EPI_BIAS_RESID_F32 = 3
WM3_EPI_QKV_ROPE = 4
WM3_EPI_GELU_GRAD_F32 = 5

_vp = ctypes.c_void_p
_i = ctypes.c_int
_f = ctypes.c_float
_ll = ctypes.c_longlong
_sz = ctypes.c_size_t


class RopeT(ctypes.Structure):
    """wm3_rope_t (include/wm3.h)."""
    _fields_ = [("dr", _vp), ("col", _vp), ("heads", _i), ("dhp", _i), ("rows", _i), ("cols", _i),
                ("period", _i), ("split", _i)]


class HaloT(ctypes.Structure):
    """wm3_halo_t (include/wm3.h)."""
    _fields_ = [("up", _vp), ("dn", _vp), ("n_up", _i), ("n_dn", _i), ("up_plane_stride", _ll),
                ("dn_plane_stride", _ll), ("up_row_off", _ll), ("dn_row_off", _ll), ("ld", _i), ("col_lo", _i)]


class BlockWeightsT(ctypes.Structure):
    """wm3_block_weights_t (include/wm3.h)."""
    _fields_ = [("ln1_g", _vp), ("ln1_b", _vp), ("w_qkv", _vp), ("b_qkv", _vp), ("w_o", _vp), ("b_o", _vp),
                ("ln2_g", _vp), ("ln2_b", _vp), ("w_1", _vp), ("b_1", _vp), ("w_2", _vp), ("b_2", _vp),
                ("hidden", _i), ("heads", _i), ("dh", _i), ("dhp", _i), ("kp", _i), ("np", _i), ("nm", _i),
                ("w_qkv_f", _vp), ("c_qkv", _vp), ("d_qkv", _vp), ("w_1_f", _vp), ("c_1", _vp), ("d_1", _vp)]


class BlockWsT(ctypes.Structure):
    """wm3_block_ws_t."""
    _fields_ = [("hn", _vp), ("qkv", _vp), ("ctx", _vp), ("mid", _vp), ("stats", _vp), ("row_stats", _vp)]


class BlockGeomT(ctypes.Structure):
    """wm3_block_geom_t."""
    _fields_ = [("batch", _i), ("depth", _i), ("rows", _i), ("cols", _i), ("rows_global", _i), ("row0", _i),
                ("halo_lo", _i), ("halo_hi", _i), ("wd", _i), ("wh", _i), ("ww", _i), ("x_prepped", _i)]


LN_SLOTS = 16  # WM3_LN_SLOTS


class LnFoldT(ctypes.Structure):
    """wm3_ln_fold_t (include/wm3.h)."""
    _fields_ = [("xh_out", _vp), ("ld_xh", _i), ("stats_out", _vp), ("row_stats", _vp), ("fold_c", _vp)]


# name -> argtypes; every function returns int status
SIGNATURES = {
    "wm3_neighbor_table": [_i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "wm3_layernorm_bf16": [_vp, _i, _i, _i, _vp, _vp, _f, _vp, _i, _vp],
    "wm3_linear": [_vp, _i, _vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, ctypes.POINTER(RopeT), _vp],
    "wm3_linear_planes": [_vp, _i, _vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, ctypes.POINTER(RopeT),
                          _i, _i, ctypes.c_longlong, _i, _vp],
    "wm3_linear_fold": [_vp, _i, _vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, ctypes.POINTER(RopeT),
                        _i, _i, ctypes.c_longlong, _i, ctypes.POINTER(HaloT), ctypes.POINTER(LnFoldT), _vp],
    "wm3_ln_fold_prep": [_vp, _i, _i, _i, _vp, _i, _f, _vp, _vp],
    "wm3_ln_fold_finalize": [_vp, _i, _i, _f, _i, _vp, _vp],
    "wm3_linear_planes_halo": [_vp, _i, _vp, _i, _i, _i, _i, _i, _vp, _i, _i, _vp, ctypes.POINTER(RopeT),
                               _i, _i, ctypes.c_longlong, _i, ctypes.POINTER(HaloT), _vp],
    "wm3_halo_signal": [_vp, _vp, _i, _vp],
    "wm3_halo_wait": [_vp, _i, _i, _vp],
    "wm3_block_qkv": [_vp, ctypes.POINTER(BlockWeightsT), ctypes.POINTER(BlockWsT), ctypes.POINTER(BlockGeomT),
                      ctypes.POINTER(RopeT), ctypes.POINTER(HaloT), _vp],
    "wm3_block_rest": [_vp, ctypes.POINTER(BlockWeightsT), ctypes.POINTER(BlockWsT), ctypes.POINTER(BlockGeomT), _vp],
    "wm3_block_na_rows": [ctypes.POINTER(BlockWeightsT), ctypes.POINTER(BlockWsT), ctypes.POINTER(BlockGeomT), _i, _i,
                          _vp],
    "wm3_block_out": [_vp, ctypes.POINTER(BlockWeightsT), ctypes.POINTER(BlockWsT), ctypes.POINTER(BlockGeomT), _vp],
    "wm3_block_fwd": [_vp, ctypes.POINTER(BlockWeightsT), ctypes.POINTER(BlockWsT), ctypes.POINTER(BlockGeomT),
                      ctypes.POINTER(RopeT), _vp],
    "wm3_natten_fwd": [_vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _f, _vp],
    "wm3_natten_fwd_rows": [_vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _f, _i, _i, _vp],
    "wm3_natten_windows": [_i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "wm3_conv_bn": [_i],
    "wm3_conv": [_i, _vp, _i, _i, _i, _i, _vp, _i, _vp, _i, _vp, _i, _i, _vp, _i, _ll, _ll, _ll, _i, _vp],
    "wm3_fields_to_nhwc": [_vp, _ll, _ll, _ll, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp],
    "wm3_tokens_to_nhwc": [_vp, _i, _i, _i, _i, _i, _vp, _vp],
    "wm3_sq_err_rows": [_i, _vp, _ll, _i, _vp, _vp, _i, _i, _i, _vp, _vp],
    "wm3_bw_amax": [_vp, _i, _i, _i, _vp, _vp],
    "wm3_bw_cast": [_vp, _i, _i, _i, _i, _vp, _i, _i, _vp, _vp],
    "wm3_bw_colsum": [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp],
    "wm3_bw_gelu": [_vp, _i, _vp, _i, _vp, _i, _i, _vp, _vp, _i, _vp],
    "wm3_bw_gelu_fwd": [_vp, _i, _vp, _i, _i, _vp, _i, _vp],
    "wm3_bw_colsum_amax": [_vp, _i, _vp, _i, _vp, _vp, _i, _i, _vp, _i, _vp, _vp, _vp, _vp],
    "wm3_bw_layernorm": [_vp, _i, _i, _i, _f, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "wm3_bw_natten": [_vp, _i, _vp, _vp, _vp, _i, _i, _i, _i, _f, _vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp],
    "wm3_bw_cast_colsum": [_vp, _i, _i, _i, _vp, _i, _vp, _vp, _vp, _vp],
    "wm3_bw_rope_q": [_vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "wm3_bw_rope": [_vp, _i, _i, _i, _i, _vp, _vp, _vp],
    "wm3_linear_gelu_grad": [_vp, _i, _vp, _i, _i, _i, _i, _vp, _i, _vp, _vp, _vp, _vp],
    "wm3_linear_tn_split_count": [_i, _i, _i],
    "wm3_linear_tn_split": [_vp, _i, _vp, _i, _i, _i, _i, _vp, _i, _vp, _sz, _vp],
    "wm3_linear_tn": [_vp, _i, _vp, _i, _i, _i, _i, _vp, _i, _vp],
    "wm3_bw_na_prep": [_vp, _i, _i, _i, _i, _vp, _i, _vp, _f, _vp, _i, _vp, _vp, _vp],
    "wm3_natten_fwd_lse": [_vp, _i, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _f, _vp, _vp],
    "wm3_natten_bwd_info": [_i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "wm3_natten_slot_table": [_i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "wm3_natten_bwd": [_vp, _i, _vp, _i, _vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i,
                       _i, _i, _i, _f, _vp],
    "wm3_zonal_power": [_i, _vp, _ll, _i, _i, _i, _i, _vp, _vp],
}

WM3_CONV_S1, WM3_CONV_S2, WM3_CONV_T2 = 0, 1, 2
WM3_CONV_OUT_NHWC, WM3_CONV_OUT_TOKENS, WM3_CONV_OUT_FIELD = 0, 1, 2


def exported_symbols() -> list[str]:
    """Every symbol include/wm3.h declares (checked against the .so by the CPU test suite)."""
    return ["wm3_last_error", "wm3_version", "wm3_sm_count", "wm3_operand_dtype"] + list(SIGNATURES)


@lru_cache(maxsize=1)
def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(
            f"libwm3.so not built at {path}; run `make` (or __graft_entry__.build()) first")
    lib = ctypes.CDLL(path)
    lib.wm3_last_error.restype = ctypes.c_char_p
    lib.wm3_last_error.argtypes = []
    lib.wm3_version.restype = _i
    lib.wm3_sm_count.restype = _i
    lib.wm3_operand_dtype.restype = _i
    lib.wm3_operand_dtype.argtypes = []
    want = {torch.float16: WM3_DTYPE_F16, torch.bfloat16: WM3_DTYPE_BF16}[ELEM]
    if lib.wm3_operand_dtype() != want:
        raise RuntimeError(f"{path} is built for operand dtype {lib.wm3_operand_dtype()}, the host layer expects "
                           f"{want} ({ELEM}); rebuild with the matching WM3_OPERAND_BF16 setting")
    for name, argt in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = _i
    return lib


def lib() -> ctypes.CDLL:
    if not torch.cuda.is_available():
        raise RuntimeError("the WM-3 B200 path needs a CUDA device; there is no CPU fallback")
    return load_library()


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load_library().wm3_last_error().decode(errors="replace")
        raise RuntimeError(f"{what}: {msg}")


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
