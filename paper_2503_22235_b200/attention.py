"""Operator-level drop-in for gridcast.attention (attention.py): natten_block and helpers.

`natten_block(x, params, prefix, extents, window, heads)` has the reference signature and error behaviour
(ConfigError before any launch, attention.py:150-155 and grid.py:98-99,119-120) and returns a new Tensor;
the input is never mutated.  The compute is the 7-launch device chain of blocks.block_forward.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib, ops
from .blocks import rope_axis_tables
from .errors import ConfigError
from .params import block_param_names, init_block_params  # noqa: F401  (re-exported API)
from .runtime import CACHE
from .tensor import payload, Tensor, host_array

__all__ = ["natten_block", "NattenBlockStream", "attention_weights", "rotary_tables", "apply_rotary",
           "init_block_params", "block_param_names", "to_device_f32", "validate_block_args"]


def to_device_f32(x) -> torch.Tensor:
    """A fresh fp32 CUDA copy of x (our Tensor, anything with .values, numpy array or torch tensor)."""
    if isinstance(x, Tensor) and x.device is not None:
        src = x.device
    elif isinstance(x, torch.Tensor):
        src = x
    else:
        v = np.asarray(payload(x))
        if v.nbytes >= (1 << 22):  # large host arrays: cast into page-locked memory, one fast upload
            h = torch.empty(v.shape, dtype=torch.float32, pin_memory=True)
            np.copyto(h.numpy(), v, casting="unsafe")
            return h.to(device="cuda").contiguous()
        src = torch.from_numpy(np.ascontiguousarray(host_array(x, np.float32)))
    return src.to(device="cuda", dtype=torch.float32, copy=True).contiguous()


def validate_block_args(shape, extents, window, heads: int) -> int:
    """attention.py:150-159 checks, in order; returns the head dim."""
    t, dim = shape
    d, h, w = (int(e) for e in extents)
    if t != d * h * w:
        raise ConfigError(f"token count {t} != prod of extents {tuple(extents)}")
    if dim % heads:
        raise ConfigError(f"dim {dim} not divisible by heads {heads}")
    for win, ext in zip(window, (d, h, w)):
        if win > ext:
            raise ConfigError(f"window {win} exceeds axis extent {ext}")
    dh = dim // heads
    if dh % 2:
        raise ConfigError(f"rotary head dim must be even, got {dh}")
    if dh // 2 < 3:
        raise ConfigError(f"head dim {dh} leaves fewer than one rotary pair per axis")
    return dh


def _foreign_tensor(x) -> bool:
    """x is a tensor of another package with the reference's surface (gridcast.autodiff.Tensor: `.values`
    plus the tape), not ours, not a torch tensor, not a plain array."""
    return (not isinstance(x, (Tensor, torch.Tensor, np.ndarray)) and hasattr(x, "values")
            and hasattr(type(x), "reshape"))


def _wrap_foreign(x, values: np.ndarray, params: dict, prefix: str, extents, window, heads: int):
    """The block output as the caller's tensor class.  For the reference's Tensor it goes through the
    reference's own recorder (autodiff.py:288-291), so grad mode and requires_grad propagate exactly as for
    the reference block.  The recorded rule is the B200 block VJP (backward.block_vjp: the block input is the
    one saved array, the intermediates are recomputed on the device), accumulating the input and every
    parameter gradient through the reference's own accumulator."""
    import sys
    record = getattr(sys.modules.get(type(x).__module__), "_record", None)
    if record is None:
        return type(x)(values)
    names = [n for n in block_param_names(prefix) if n in params]
    parents = [x] + [params[n] for n in names]
    ext, win = tuple(int(e) for e in extents), tuple(int(w) for w in window)

    def rule(g, saved, add):
        from .backward import block_vjp
        (xv,) = saved
        gx, grads = block_vjp(xv, params, prefix, ext, win, heads, g)
        add(x, gx)
        for n in names:
            add(params[n], grads[n])

    return record("natten_block_b200", values, parents, [x.values], rule)


def natten_block(x, params: dict, prefix: str, extents, window, heads: int):
    """One pre-norm neighborhood attention block (attention.py:146-184) on the B200.

    Returns our Tensor (device-backed) for our / torch / numpy inputs.  Given the reference's own Tensor
    (the operator-level seam: `gridcast.model.natten_block = natten_block`), it returns a
    tensor of the caller's class built from the float64 result, so the reference's encode / process / decode
    keep applying their own ops (`tokens.reshape(...)`, model.py:357-360) to it.  It is recorded on the
    reference's tape like the reference block, with the B200 block VJP as its backward rule (backward.py), so
    the reference's training, checkpointing and offload engine run the block forward and backward on the
    device."""
    shape = tuple(x.shape)
    dh = validate_block_args(shape, extents, window, heads)
    foreign = _foreign_tensor(x)
    bw = CACHE.block(params, prefix, heads)
    if bw.hidden != shape[1]:
        raise ConfigError(f"parameters {prefix} have width {bw.hidden}, tokens have {shape[1]}")
    xd = to_device_f32(x)
    from .blocks import block_forward
    block_forward(xd, bw, CACHE.workspace(extents, window, bw), CACHE.rope(extents, dh), tuple(extents),
                  tuple(window))
    if foreign:
        from .tensor import device_to_host_f64
        return _wrap_foreign(x, device_to_host_f64(xd), params, prefix, extents, window, heads)
    return Tensor(device=xd)


class NattenBlockStream:
    """natten_block over a stream of host token batches, with the transfers overlapped (serving path).

    `submit(host_in, host_out)` takes page-locked float32 (T, dim) host tensors and returns at once: the batch is
    copied host->device on one CUDA stream, the block runs on a second, the result is copied device->host on a
    third, so batch i+1's upload and batch i-1's download run under batch i's compute (both PCIe directions at
    once).  Three device buffers rotate, so an upload never waits for the download of the batch just before
    (with two, upload i+1 waits for download i-1 and the period is (up + compute + down) / 2 instead of the
    transfer time); `synchronize()` waits for everything submitted.  Each batch's result equals
    natten_block(host_in, ...) bitwise (same kernels, same inputs)."""

    NBUF = 3

    def __init__(self, params: dict, prefix: str, extents, window, heads: int, dim: int):
        t = int(np.prod(extents))
        self.dh = validate_block_args((t, dim), extents, window, heads)
        self.extents, self.window = tuple(int(e) for e in extents), tuple(int(e) for e in window)
        self.bw = CACHE.block(params, prefix, heads)
        # a private workspace: two streams (e.g. a pipeline of two blocks) run concurrently on their own
        # s_run streams and must not share the q/k/v / ctx / MLP buffers
        from .blocks import Workspace
        self.ws = Workspace(ops.KVGrid(self.extents, self.window), self.bw)
        self.rope = CACHE.rope(self.extents, self.dh)
        self.buf = [torch.empty((t, dim), dtype=torch.float32, device="cuda") for _ in range(self.NBUF)]
        self.s_in, self.s_run, self.s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.uploaded = [torch.cuda.Event() for _ in range(self.NBUF)]
        self.computed = [torch.cuda.Event() for _ in range(self.NBUF)]
        self.downloaded = [None] * self.NBUF
        self.i = 0
        # weight conversion, workspace zero-fill and rotary tables were queued on the creating stream: finish
        # them before s_run (which only waits on uploads) can read them
        torch.cuda.current_stream().synchronize()

    def submit(self, host_in: torch.Tensor, host_out: torch.Tensor) -> None:
        from .blocks import block_forward
        b = self.i % self.NBUF
        self.i += 1
        dev = self.buf[b]
        with torch.cuda.stream(self.s_in):
            if self.downloaded[b] is not None:  # the download of the batch that last used this buffer
                self.s_in.wait_event(self.downloaded[b])
            dev.copy_(host_in, non_blocking=True)
            self.uploaded[b].record(self.s_in)
        with torch.cuda.stream(self.s_run):
            self.s_run.wait_event(self.uploaded[b])
            block_forward(dev, self.bw, self.ws, self.rope, self.extents, self.window)
            self.computed[b].record(self.s_run)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.computed[b])
            host_out.copy_(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.s_out)
            self.downloaded[b] = ev

    def synchronize(self) -> None:
        for s in (self.s_in, self.s_run, self.s_out):
            s.synchronize()


def attention_weights(x_values, params: dict, prefix: str, extents, window, heads: int) -> np.ndarray:
    """Softmax weights (T, heads, K) for inspection (attention.py:187-212), produced by the fused attention
    kernel itself.

    q and k come from the block's own LN + QKV/rotary kernels.  The probabilities are read out of the NA kernel
    by feeding it one-hot values: in pass r, V of token r * dhp + j is the unit vector e_j (every head) and
    every other token's V is 0, so the kernel's normalised output row of query t is exactly its softmax weight
    on each key of that token range (its own masked online softmax, fp32 statistics, operand-rounded output).
    ceil(T / dhp) passes cover every key; the weights are then gathered in window order with the kernel's
    neighbor table (grid.py:124-127 K order)."""
    xd = to_device_f32(x_values)
    t, dim = xd.shape
    dh = validate_block_args((t, dim), extents, window, heads)
    extents, window = tuple(int(e) for e in extents), tuple(int(e) for e in window)
    bw = CACHE.block(params, prefix, heads)
    ws = CACHE.workspace(extents, window, bw)
    rope = CACHE.rope(extents, dh)
    ops.layernorm_bf16(xd, bw.ln1_g, bw.ln1_b, out=ws.hn)
    ops.linear_grid(ws.hn, bw.w_qkv, _lib.WM3_EPI_QKV_ROPE, bw.b_qkv, ws.qkv, ws.grid,
                    rope=rope.struct(extents, 0, bw.heads, bw.dhp))
    dhp, sec = bw.dhp, heads * bw.dhp
    qkv = ws.qkv.clone()  # single band, no halos: grid rows are tokens
    v = qkv[:, 2 * sec:].view(t, heads, dhp)
    full = torch.empty((t, heads, t), dtype=torch.float32, device=xd.device)
    for r0 in range(0, t, dhp):
        n = min(dhp, t - r0)
        v.zero_()
        idx = torch.arange(n, device=xd.device)
        v[r0 + idx, :, idx] = 1.0
        out = ops.natten(qkv, ws.grid, heads, dhp, dh, window).view(t, heads, dhp)
        full[:, :, r0:r0 + n] = out[:, :, :n].float()
    table = ops.neighbor_table(extents, window)  # (T, K)
    probs = torch.gather(full, 2, table.unsqueeze(1).expand(t, heads, table.shape[1]))
    return probs.double().cpu().numpy()


def rotary_tables(extents, head_dim: int):
    """cos/sin (T, 1, head_dim // 2) float64 (attention.py:48-84), assembled from the per-axis tables."""
    d, h, w = (int(e) for e in extents)
    n = head_dim // 2
    rope_axis_tables(extents, head_dim)  # same validation as the device tables
    di, hi, wi = np.unravel_index(np.arange(d * h * w), (d, h, w))
    from .blocks import _wavelengths, pair_split
    pd, pr, pc = pair_split(n)
    ang = np.empty((d * h * w, n))
    ang[:, :pd] = 2.0 * math.pi * di[:, None] / _wavelengths(d, pd)[None, :]
    ang[:, pd:pd + pr] = 2.0 * math.pi * hi[:, None] / _wavelengths(h, pr)[None, :]
    ang[:, pd + pr:] = 2.0 * math.pi * wi[:, None] * np.arange(1, pc + 1)[None, :] / w
    return np.ascontiguousarray(np.cos(ang)[:, None, :]), np.ascontiguousarray(np.sin(ang)[:, None, :])


def apply_rotary(x, cos, sin):
    """Rotate feature pairs (j, j + dh/2) of x (T, heads, dh) by per-token phases (attention.py:87-92)."""
    xv, cv, sv = host_array(x), host_array(cos), host_array(sin)
    half = xv.shape[-1] // 2
    a, b = xv[..., :half], xv[..., half:]
    return Tensor(np.concatenate([a * cv - b * sv, a * sv + b * cv], axis=-1))
