"""Encoder / decoder convolution pyramids on the device (model.py:296-360, 363-421).

Weights are converted once per parameter set into the implicit-GEMM layout of csrc/conv.cu; activations
live in padded bf16 NHWC buffers ([imgs][H + 2][W + 2][Cp], zero halo rows, wrapped halo columns) that are
allocated once per configuration and reused.  All depth planes go through the shared pyramid weights as the
images of one launch per conv (model.py:384,417).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .config import DOWNSAMPLE_STAGES, N_STATIC_FIELDS, ModelConfig
from .errors import ConfigError
from .tensor import host_values


def cpad(c: int) -> int:
    return (c + 63) // 64 * 64


def conv_bn(cout: int) -> int:
    """N tile of the conv kernel for `cout` output channels (csrc/conv.cu wm3_conv_bn)."""
    return 64 if cout <= 64 else (128 if cout <= 128 else (192 if cout <= 192 else 256))


@dataclass
class ConvW:
    mode: int
    cin: int
    cinp: int
    cout: int
    w: torch.Tensor   # bf16 K-major, see include/wm3.h
    b: torch.Tensor   # fp32 [cout_pad]


def conv3_weights(w: np.ndarray, b: np.ndarray, stride: int, device="cuda") -> ConvW:
    """(Cout, Cin, 3, 3) -> [cout_pad][tap = kh*3 + kw][cinp]."""
    cout, cin = w.shape[:2]
    cinp = cpad(cin)
    cp = (cout + conv_bn(cout) - 1) // conv_bn(cout) * conv_bn(cout)
    buf = np.zeros((cp, 9, cinp), dtype=np.float32)
    buf[:cout, :, :cin] = w.transpose(0, 2, 3, 1).reshape(cout, 9, cin)
    bias = np.zeros(cp, dtype=np.float32)
    bias[:cout] = b
    mode = _lib.WM3_CONV_S1 if stride == 1 else _lib.WM3_CONV_S2
    return ConvW(mode, cin, cinp, cout, torch.from_numpy(buf.reshape(cp, -1)).to(device, _lib.ELEM),
                 torch.from_numpy(bias).to(device))


def convT_weights(w: np.ndarray, b: np.ndarray, device="cuda") -> ConvW:
    """(Cin, Cout, 4, 4) -> [class 2a + b][cout_pad][tap 2tr + tc][cinp] = W[:, :, 3-a-2tr, 3-b-2tc]^T."""
    cin, cout = w.shape[:2]
    cinp = cpad(cin)
    cp = (cout + conv_bn(cout) - 1) // conv_bn(cout) * conv_bn(cout)
    buf = np.zeros((4, cp, 4, cinp), dtype=np.float32)
    for a in range(2):
        for bb in range(2):
            for tr in range(2):
                for tc in range(2):
                    buf[2 * a + bb, :cout, 2 * tr + tc, :cin] = w[:, :, 3 - a - 2 * tr, 3 - bb - 2 * tc].T
    bias = np.zeros(cp, dtype=np.float32)
    bias[:cout] = b
    return ConvW(_lib.WM3_CONV_T2, cin, cinp, cout, torch.from_numpy(buf.reshape(4 * cp, -1)).to(device,
                                                                                                 _lib.ELEM),
                 torch.from_numpy(bias).to(device))


def _pw(params, name):
    return host_values(params[name + ".w"]), host_values(params[name + ".b"])


def nhwc(imgs: int, h: int, w: int, c: int, device="cuda") -> torch.Tensor:
    return torch.zeros((imgs, h + 2, w + 2, cpad(c)), dtype=_lib.ELEM, device=device)


# Measurement hook (bench.py / tools/encdec_roofline.py): when set, called as hook(cw, imgs, h, w, phase) with
# phase "begin" / "end" around every conv launch on the current stream (e.g. to record CUDA events).
CONV_HOOK = None


def conv_layer_flops(cw: ConvW, imgs: int, h: int, w: int) -> float:
    """Algorithmic FLOPs of one run_conv call (h, w = input extents as passed to run_conv)."""
    if cw.mode == _lib.WM3_CONV_S1:
        return 2.0 * imgs * h * w * cw.cout * 9 * cw.cin
    if cw.mode == _lib.WM3_CONV_S2:
        return 2.0 * imgs * (h // 2) * (w // 2) * cw.cout * 9 * cw.cin
    return 2.0 * imgs * (2 * h) * (2 * w) * cw.cout * 4 * cw.cin


def run_conv(cw: ConvW, x: torch.Tensor, imgs: int, h: int, w: int, out: torch.Tensor, *, gelu: bool = False,
             resid: torch.Tensor | None = None, kind: int = _lib.WM3_CONV_OUT_NHWC, img_stride: int = 0,
             a_stride: int = 0, p_stride: int = 0, chan_div: int = 1) -> torch.Tensor:
    """One implicit-GEMM conv launch: x padded NHWC (imgs, h+2, w+2, cinp) -> out (layout per `kind`)."""
    if x.shape[-1] != cw.cinp:
        raise RuntimeError(f"conv input has {x.shape[-1]} channels, weights expect {cw.cinp}")
    out_cp = out.shape[-1] if kind == _lib.WM3_CONV_OUT_NHWC else 0
    resid_cp = resid.shape[-1] if resid is not None else 0
    if CONV_HOOK is not None:
        CONV_HOOK(cw, imgs, h, w, "begin")
    check(_lib.lib().wm3_conv(cw.mode, ptr(x), imgs, h, w, cw.cinp, ptr(cw.w), cw.cout, ptr(cw.b), int(gelu),
                              ptr(resid), resid_cp, kind, ptr(out), out_cp, img_stride, a_stride, p_stride,
                              chan_div, stream_ptr()), "wm3_conv")
    if CONV_HOOK is not None:
        CONV_HOOK(cw, imgs, h, w, "end")
    return out


def fields_to_nhwc(src: torch.Tensor, imgs: int, channels: int, h: int, w: int, dst: torch.Tensor,
                   img_stride: int, a_stride: int, p_stride: int, chan_div: int,
                   overflow: torch.Tensor | None = None) -> None:
    check(_lib.lib().wm3_fields_to_nhwc(ptr(src), img_stride, a_stride, p_stride, chan_div, imgs, channels, h, w,
                                        dst.shape[-1], ptr(dst), ptr(overflow), stream_ptr()), "wm3_fields_to_nhwc")


def check_input_range(bufs: "PyramidBuffers") -> None:
    """Raise ConfigError if the last encode_planes saw an input value the 16-bit operand type cannot hold
    (|x| > 65504 for fp16, or a non-finite value): the reference accepts any float64 magnitude, the B200 path
    refuses instead of convolving infinities.  One device->host read of a flag (synchronises the stream)."""
    if int(bufs.overflow.item()):
        lim = "65504 (fp16 operands)" if _lib.ELEM == torch.float16 else "the bf16 range"
        raise ConfigError(f"input fields hold values beyond {lim} or non-finite values; standardise the fields "
                          f"before encoding")


def tokens_to_nhwc(tokens: torch.Tensor, imgs: int, h: int, w: int, dst: torch.Tensor) -> None:
    check(_lib.lib().wm3_tokens_to_nhwc(ptr(tokens), imgs, h, w, tokens.shape[-1], dst.shape[-1], ptr(dst),
                                        stream_ptr()), "wm3_tokens_to_nhwc")


# ------------------------------------------------------------------------------------------------
# weights
# ------------------------------------------------------------------------------------------------
@dataclass
class StageW:
    resample: ConvW
    res: list  # [(conv1, conv2), (conv1, conv2)]


def _res(params, prefix):
    return [(conv3_weights(*_pw(params, f"{prefix}.res{j}.conv1"), 1),
             conv3_weights(*_pw(params, f"{prefix}.res{j}.conv2"), 1)) for j in range(2)]


class EncoderWeights:
    def __init__(self, params: dict, prefix: str):
        self.stem_sfc = conv3_weights(*_pw(params, f"{prefix}.stem_sfc"), 1)
        self.stem_atm = conv3_weights(*_pw(params, f"{prefix}.stem_atm"), 1)
        self.stages = [StageW(conv3_weights(*_pw(params, f"{prefix}.stage{i}.down"), 2), _res(params,
                                                                                             f"{prefix}.stage{i}"))
                       for i in range(DOWNSAMPLE_STAGES)]


class DecoderWeights:
    def __init__(self, params: dict):
        self.stages = [StageW(convT_weights(*_pw(params, f"dec.stage{i}.up")), _res(params, f"dec.stage{i}"))
                       for i in range(DOWNSAMPLE_STAGES)]
        self.head_sfc = conv3_weights(*_pw(params, "dec.head_sfc"), 1)
        self.head_atm = conv3_weights(*_pw(params, "dec.head_atm"), 1)


# ------------------------------------------------------------------------------------------------
# activations
# ------------------------------------------------------------------------------------------------
class PyramidBuffers:
    """Ping-pong padded NHWC buffers for every pyramid level of one configuration (D images)."""

    def __init__(self, cfg: ModelConfig, device="cuda"):
        g = cfg.grid
        d = cfg.depth_planes
        self.cfg = cfg
        self.levels = []
        chans = [cfg.stem_channels] + list(cfg.stage_channels)
        for i in range(DOWNSAMPLE_STAGES + 1):
            h, w = g.rows >> i, g.cols >> i
            enc_c = chans[i]
            dec_c = ([cfg.stem_channels] + list(cfg.stage_channels[:-1]))[i] if i < DOWNSAMPLE_STAGES else cfg.hidden
            c = max(enc_c, dec_c)
            self.levels.append((h, w, [nhwc(d, h, w, c, device) for _ in range(3)]))
        # encoder inputs: surface + statics (one image) and folded atmosphere (level groups)
        self.sfc_in = torch.zeros((cfg.surface_in + N_STATIC_FIELDS, g.rows, g.cols), dtype=torch.float32,
                                  device=device)
        self.atm_in = torch.zeros((cfg.atmos_vars, cfg.levels, g.rows, g.cols), dtype=torch.float32, device=device)
        self.in_sfc = nhwc(1, g.rows, g.cols, cfg.surface_in + N_STATIC_FIELDS, device)
        self.in_atm = nhwc(cfg.levels // cfg.level_patch, g.rows, g.cols, cfg.atmos_vars * cfg.level_patch, device)
        self.statics_ready = False
        self.overflow = torch.zeros(1, dtype=torch.int32, device=device)  # fields_to_nhwc range flag

    def buf(self, level: int, k: int, c: int) -> torch.Tensor:
        b = self.levels[level][2][k]
        if b.shape[-1] != cpad(c):  # halo rows must stay zero: never reinterpret a buffer's pitch
            raise ConfigError(f"pyramid level {level} holds {b.shape[-1]} channels, asked for {c}")
        return b


def _res_block(ws: StageW, bufs: PyramidBuffers, level: int, x_idx: int, imgs: int, h: int, w: int, c: int,
               lo: int = 0) -> int:
    """Two res blocks x + conv2(gelu(conv1(x))) (model.py:304-306) with ping-pong buffers on images
    [lo, lo + imgs); returns result idx."""
    for conv1, conv2 in ws.res:
        t_idx, y_idx = [k for k in range(3) if k != x_idx][:2]
        x = bufs.buf(level, x_idx, c)[lo:lo + imgs]
        t = bufs.buf(level, t_idx, c)[lo:lo + imgs]
        y = bufs.buf(level, y_idx, c)[lo:lo + imgs]
        run_conv(conv1, x, imgs, h, w, t, gelu=True)
        run_conv(conv2, t, imgs, h, w, y, resid=x)
        x_idx = y_idx
    return x_idx


# encoder stages run plane by plane while the host fields upload (encode_planes with before_plane)
PER_PLANE_STAGES = 2


def encode_planes(ew: EncoderWeights, bufs: PyramidBuffers, cfg: ModelConfig, tokens_out: torch.Tensor,
                  planes: tuple[int, int] | None = None, before_plane=None) -> None:
    """bufs.sfc_in / atm_in (device fp32) -> latent tokens (D*h*w, hidden) fp32.

    planes = (lo, hi) encodes only depth planes [lo, hi) (plane 0 = surface, p >= 1 = atmosphere level group
    p - 1) into their token rows: the planes share the pyramid weights and never interact before the encoder
    blocks, so the split is exact (bands.forecast_banded runs one range per rank).
    before_plane(q): with it, the input layout copy, the stem convolution and the first PER_PLANE_STAGES stages
    run plane by plane, each plane after before_plane(q) (model.encode: make the stream wait for that plane's
    host upload), so the upload of plane q + 1 overlaps the convolutions of plane q; the per-plane launches write
    the same bytes as the batched ones."""
    g = cfg.grid
    hh, ww = g.rows, g.cols
    d = cfg.depth_planes
    lo, hi = (0, d) if planes is None else (int(planes[0]), int(planes[1]))
    if not 0 <= lo < hi <= d:
        raise ConfigError(f"plane range {planes} outside [0, {d})")
    n = hi - lo
    csfc = cfg.surface_in + N_STATIC_FIELDS
    catm = cfg.atmos_vars * cfg.level_patch
    hw = hh * ww
    x0 = bufs.buf(0, 0, cfg.stem_channels)
    bufs.overflow.zero_()
    def stems(a: int, b: int) -> None:  # input layout + stem conv of planes [a, b)
        if a == 0:
            fields_to_nhwc(bufs.sfc_in, 1, csfc, hh, ww, bufs.in_sfc, 0, hw, 0, 1, bufs.overflow)
            run_conv(ew.stem_sfc, bufs.in_sfc, 1, hh, ww, x0[0:1])
        a0 = max(a, 1)
        if b > a0:  # atmosphere level groups a0 - 1 .. b - 2
            fields_to_nhwc(bufs.atm_in.view(-1)[(a0 - 1) * cfg.level_patch * hw:], b - a0, catm, hh, ww,
                           bufs.in_atm[a0 - 1:b - 1], cfg.level_patch * hw, cfg.levels * hw, hw, cfg.level_patch,
                           bufs.overflow)
            run_conv(ew.stem_atm, bufs.in_atm[a0 - 1:b - 1], b - a0, hh, ww, x0[a0:b])

    x_idx, c = 0, cfg.stem_channels
    first = 0
    if before_plane is None:
        stems(lo, hi)
    elif DOWNSAMPLE_STAGES > 1:
        # per plane: stem and the first PER_PLANE_STAGES stages (not the token-writing last one), while the next
        # plane uploads — a plane's stem + two stages take longer than its upload, so only the first plane's
        # upload is exposed
        first = min(PER_PLANE_STAGES, DOWNSAMPLE_STAGES - 1)
        for q in range(lo, hi):
            before_plane(q)
            stems(q, q + 1)
            xi, ci = 0, cfg.stem_channels
            for i in range(first):
                st = ew.stages[i]
                h2, w2 = hh >> (i + 1), ww >> (i + 1)
                c_out = cfg.stage_channels[i]
                run_conv(st.resample, bufs.buf(i, xi, ci)[q:q + 1], 1, h2 * 2, w2 * 2, bufs.buf(i + 1, 0, c_out)[q:q + 1])
                xi, ci = _res_block(st, bufs, i + 1, 0, 1, h2, w2, c_out, q), c_out
        x_idx, c = xi, ci
    else:
        for q in range(lo, hi):
            before_plane(q)
            stems(q, q + 1)
    for i, st in enumerate(ew.stages):
        if i < first:
            continue
        h2, w2 = hh >> (i + 1), ww >> (i + 1)
        c_out = cfg.stage_channels[i]
        last = i == DOWNSAMPLE_STAGES - 1
        y = bufs.buf(i + 1, 0, c_out)[lo:hi]
        run_conv(st.resample, bufs.buf(i, x_idx, c)[lo:hi], n, h2 * 2, w2 * 2, y)
        x_idx = 0
        if not last:
            x_idx = _res_block(st, bufs, i + 1, x_idx, n, h2, w2, c_out, lo)
        else:
            # final res block writes the fp32 token grid directly (model.py:350-354)
            conv1, conv2 = st.res[0]
            t, z = bufs.buf(i + 1, 1, c_out)[lo:hi], bufs.buf(i + 1, 2, c_out)[lo:hi]
            run_conv(conv1, y, n, h2, w2, t, gelu=True)
            run_conv(conv2, t, n, h2, w2, z, resid=y)
            conv1, conv2 = st.res[1]
            run_conv(conv1, z, n, h2, w2, t, gelu=True)
            run_conv(conv2, t, n, h2, w2, tokens_out[lo * h2 * w2:hi * h2 * w2], resid=z,
                     kind=_lib.WM3_CONV_OUT_TOKENS)
            # residual add for the token output happens in-kernel from the padded skip buffer
        c = c_out


def decode_planes(dw: DecoderWeights, bufs: PyramidBuffers, cfg: ModelConfig, tokens: torch.Tensor,
                  surface_out: torch.Tensor, atmos_out: torch.Tensor, planes: tuple[int, int] | None = None,
                  on_plane=None) -> None:
    """latent tokens (fp32) -> surface (surface_out, H, W) and atmos (A, L, H, W) fp32 fields.

    planes = (lo, hi): only depth planes [lo, hi) (surface if lo == 0, atmosphere levels of groups lo-1..hi-2)
    are decoded; the up-pyramid treats planes independently, so the split is exact.
    on_plane(q): with it, the full-resolution stage and the heads run plane by plane and on_plane(q) is called
    (on the host, after queueing) once plane q's fields are written, so a caller can stream them out while the
    next plane is convolved; the per-plane launches write the same bytes as the batched ones."""
    g = cfg.grid
    d, h, w = cfg.latent_extents
    lo, hi = (0, d) if planes is None else (int(planes[0]), int(planes[1]))
    if not 0 <= lo < hi <= d:
        raise ConfigError(f"plane range {planes} outside [0, {d})")
    n = hi - lo
    lvl = DOWNSAMPLE_STAGES
    x = bufs.buf(lvl, 0, cfg.hidden)[lo:hi]
    tokens_to_nhwc(tokens[lo * h * w:hi * h * w], n, h, w, x)
    chans = [cfg.hidden] + list(cfg.stage_channels[-2::-1]) + [cfg.stem_channels]
    hh, ww = g.rows, g.cols
    p = cfg.level_patch

    def heads(a: int, b: int, full) -> None:  # fields of planes [a, b)
        if a == 0:
            run_conv(dw.head_sfc, full[0:1], 1, hh, ww, surface_out, kind=_lib.WM3_CONV_OUT_FIELD, img_stride=0,
                     a_stride=hh * ww, p_stride=0, chan_div=1)
        a0 = max(a, 1)
        if b > a0:  # level groups a0 - 1 .. b - 2 -> levels [(a0 - 1) p, (b - 1) p)
            dst = atmos_out.view(-1)[(a0 - 1) * p * hh * ww:]
            run_conv(dw.head_atm, full[a0:b], b - a0, hh, ww, dst, kind=_lib.WM3_CONV_OUT_FIELD,
                     img_stride=p * hh * ww, a_stride=cfg.levels * hh * ww, p_stride=hh * ww, chan_div=p)

    x_idx = 0
    stages = list(enumerate(dw.stages))
    last_i = len(stages) - 1
    for i, st in stages:
        lvl_out = lvl - i - 1
        ho, wo = g.rows >> lvl_out, g.cols >> lvl_out
        if i == last_i and on_plane is not None:
            # the surface plane (smallest download) last, so the copy left after the decoder is the shortest
            for q in [q for q in range(lo, hi) if q != 0] + ([0] if lo == 0 else []):
                src = bufs.buf(lvl - i, x_idx, chans[i])[q:q + 1]
                y = bufs.buf(lvl_out, 0, chans[i + 1])[q:q + 1]
                run_conv(st.resample, src, 1, ho // 2, wo // 2, y)
                q_idx = _res_block(st, bufs, lvl_out, 0, 1, ho, wo, chans[i + 1], q)
                heads(q, q + 1, bufs.buf(0, q_idx, cfg.stem_channels))
                on_plane(q)
            return
        src = bufs.buf(lvl - i, x_idx, chans[i])[lo:hi]
        y = bufs.buf(lvl_out, 0, chans[i + 1])[lo:hi]
        run_conv(st.resample, src, n, ho // 2, wo // 2, y)
        x_idx = _res_block(st, bufs, lvl_out, 0, n, ho, wo, chans[i + 1], lo)
    heads(lo, hi, bufs.buf(0, x_idx, cfg.stem_channels))


def check_grid(cfg: ModelConfig) -> None:
    if cfg.grid.cols % (1 << DOWNSAMPLE_STAGES):
        raise ConfigError("grid columns must divide by the downsampling factor")
