"""Forecast verification on the device (gridcast/evaluation.py): weighted RMSE, zonal spectra, blur, ensembles.

Same functions, signatures, conventions and errors as the reference (evaluation.py:1-190): cos-latitude row
weights used as given with the plain cell count as divisor, mean-square zonal power, power interpolated in log
wavelength and averaged over the rows whose resolvable range covers the target, the unbounded blur sentinel,
leading-k ensemble-mean curves, percent-change scorecards.

The heavy parts run in libwm3.so (csrc/metrics.cu: float64 accumulation, fixed reduction order): the weighted
squared error per (time, row) and, for rows up to 256 columns, the per-row zonal power spectra by direct DFT,
each optionally of the mean of the leading k ensemble members computed on the fly; wider rows (the 1440-column
0.25 deg grid) take their spectra from cuFFT in float64 (torch.fft.rfft).  Inputs may be numpy arrays (copied to the device once) or
CUDA tensors (used in place: decoded forecasts and ensemble members are scored without leaving HBM); only a
(times x rows) or (rows x bins) float64 array comes back to the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr, stream_ptr
from .errors import ConfigError, DataError
from .grid import GridSpec, latitude_weights, row_circumference_km
from .tensor import host_array

__all__ = ["BLUR_UNBOUNDED", "DEFAULT_SUBSET_SIZES", "latitude_rmse", "zonal_power", "power_at_wavelength",
           "blur_index", "subset_sizes", "ensemble_curve", "scorecard", "plane_scores"]

BLUR_UNBOUNDED = float("inf")
DEFAULT_SUBSET_SIZES = (1, 2, 4, 8, 12, 16, 20, 24, 28, 32, 36, 40, 44, 48, 51)


def _device(x) -> torch.Tensor:
    """CUDA float32 / float64 contiguous view or copy of x (numpy, torch, or anything with .values / .device)."""
    dev = getattr(x, "device", None)
    if isinstance(dev, torch.Tensor):  # our Tensor wrapper with a device buffer
        x = dev
    elif not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(host_array(x, np.float64)))
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    return x.to("cuda").contiguous()


def _dtype_code(t: torch.Tensor) -> int:
    return 0 if t.dtype == torch.float32 else 1


def _time_stack(x: torch.Tensor, spec: GridSpec, name: str) -> torch.Tensor:
    if x.dim() == 2:
        x = x[None]
    if x.dim() != 3 or tuple(x.shape[1:]) != (spec.rows, spec.cols):
        raise DataError(f"{name} must be (times, {spec.rows}, {spec.cols}); got {tuple(x.shape)}")
    return x


def _weights(spec: GridSpec) -> torch.Tensor:
    return torch.from_numpy(latitude_weights(spec)).to("cuda")


def _rmse_from(members: torch.Tensor, k: int, truth: torch.Tensor, spec: GridSpec) -> float:
    """Weighted RMSE of the mean of the leading k members (members: (n, T, H, W), same dtype as truth)."""
    t = truth.shape[0]
    partial = torch.empty((t, spec.rows), dtype=torch.float64, device="cuda")
    check(_lib.lib().wm3_sq_err_rows(_dtype_code(truth), ptr(members), members[0].numel() if k > 1 else 0, int(k),
                                     ptr(truth), ptr(_weights(spec)), t, spec.rows, spec.cols, ptr(partial),
                                     stream_ptr()), "wm3_sq_err_rows")
    per_time = np.sqrt(partial.cpu().numpy().sum(axis=1) / (spec.rows * spec.cols))
    return float(per_time.mean())


def latitude_rmse(pred, truth, spec: GridSpec) -> float:
    """Cos-latitude weighted RMSE averaged over times (evaluation.py:37-52)."""
    p = _time_stack(_device(pred), spec, "pred")
    g = _time_stack(_device(truth), spec, "truth")
    if p.shape != g.shape:
        raise DataError(f"shape mismatch {tuple(p.shape)} vs {tuple(g.shape)}")
    if p.dtype != g.dtype:
        p, g = p.double(), g.double()
    return _rmse_from(p[None], 1, g, spec)


# Rows wider than this use cuFFT (torch.fft, float64: O(W log W)); narrower ones the direct-DFT kernel of
# csrc/metrics.cu (O(W^2) but one launch and exact twiddles).  At 1440 columns the direct DFT is ~100x the work.
DFT_MAX_COLS = 256


def _zonal_power_dev(fields: torch.Tensor, k: int, spec: GridSpec) -> torch.Tensor:
    """(imgs, rows, cols//2 + 1) float64 power of fields (imgs, rows, cols), or of the leading-k member mean
    when fields is (n, imgs, rows, cols) and k > 1."""
    imgs = fields.shape[-3]
    if spec.cols > DFT_MAX_COLS:
        f = fields[:k].double().mean(dim=0) if fields.dim() == 4 else fields.double()
        coef = torch.fft.rfft(f, dim=-1)
        pw = (coef.real * coef.real + coef.imag * coef.imag) / float(spec.cols * spec.cols)
        last = pw.shape[-1] - 1 if spec.cols % 2 == 0 else pw.shape[-1]
        pw[..., 1:last] *= 2.0
        return pw.contiguous()
    out = torch.empty((imgs, spec.rows, spec.cols // 2 + 1), dtype=torch.float64, device="cuda")
    stride = fields[0].numel() if k > 1 else 0
    check(_lib.lib().wm3_zonal_power(_dtype_code(fields), ptr(fields), stride, int(k), imgs, spec.rows, spec.cols,
                                     ptr(out), stream_ptr()), "wm3_zonal_power")
    return out


def zonal_power(field, spec: GridSpec) -> np.ndarray:
    """Per-row zonal power spectrum (rows, cols//2 + 1), mean-square convention (evaluation.py:59-75)."""
    f = _device(field)
    if tuple(f.shape) != (spec.rows, spec.cols):
        raise DataError(f"field must be {(spec.rows, spec.cols)}; got {tuple(f.shape)}")
    return _zonal_power_dev(f[None], 1, spec)[0].cpu().numpy()


def _interp_plan(spec: GridSpec, n_wave: int, wavelength_km: float):
    """Per-row interpolation plan for power_at_wavelength (evaluation.py:78-107): bracketing wavenumbers lo / hi
    of circumference / wavelength, the weight t of hi (linear in log(lambda) = log(circumference) - log(m), which
    is exactly np.interp on the reversed arrays), and the row weights (cos latitude, 0 for rows whose resolvable
    range misses the target)."""
    if wavelength_km <= 0:
        raise ConfigError("wavelength must be positive")
    if n_wave < 1:
        raise ConfigError("grid too narrow for any zonal wave")
    circ = row_circumference_km(spec)
    ok = (circ / n_wave <= wavelength_km) & (wavelength_km <= circ)  # lam[-1] <= target <= lam[0]
    if not ok.any():
        raise ConfigError(f"wavelength {wavelength_km} km outside every row's resolvable range")
    lo = np.clip(np.floor(circ / wavelength_km), 1, n_wave).astype(np.int64)
    hi = np.minimum(lo + 1, n_wave)
    xl, xh = np.log(circ / lo), np.log(circ / hi)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.where(hi > lo, (np.log(wavelength_km) - xl) / (xh - xl), 0.0)
    wr = np.where(ok, latitude_weights(spec), 0.0)
    return lo, hi, t, wr / wr.sum()


def _interp_rows(p, spec: GridSpec, wavelength_km: float):
    """Power at one wavelength from (..., rows, bins) spectra (numpy or CUDA tensor), vectorised over rows and
    leading planes; a float for 2D input, an array over the leading dimensions otherwise."""
    lo, hi, t, wr = _interp_plan(spec, p.shape[-1] - 1, wavelength_km)
    rows = np.arange(spec.rows)
    if isinstance(p, torch.Tensor):  # on the device: only the per-plane values come back
        dev = p.device
        rows_t, lo_t, hi_t = (torch.from_numpy(a).to(dev) for a in (rows, lo, hi))
        t_t, w_t = torch.from_numpy(t).to(dev), torch.from_numpy(wr).to(dev)
        plo, phi = p[..., rows_t, lo_t], p[..., rows_t, hi_t]
        return ((plo + (phi - plo) * t_t) * w_t).sum(dim=-1).cpu().numpy()
    plo, phi = p[..., rows, lo], p[..., rows, hi]
    return ((plo + (phi - plo) * t) * wr).sum(axis=-1)


def power_at_wavelength(field, spec: GridSpec, wavelength_km: float) -> float:
    if wavelength_km <= 0:
        raise ConfigError("wavelength must be positive")
    return float(_interp_rows(zonal_power(field, spec), spec, wavelength_km))


def _blur_from_powers(pf: float, pt: float) -> float:
    if pt <= 0.0:
        return BLUR_UNBOUNDED
    ratio = pf / pt
    if ratio <= 0.0:
        return BLUR_UNBOUNDED
    return float(1.0 / np.sqrt(ratio))


def blur_index(pred, truth, spec: GridSpec, wavelength_km: float) -> float:
    """1 / sqrt(power ratio pred / truth) at one wavelength; the unbounded sentinel when undefined
    (evaluation.py:110-127)."""
    pt = power_at_wavelength(truth, spec, wavelength_km)
    pf = power_at_wavelength(pred, spec, wavelength_km)
    return _blur_from_powers(pf, pt)


def subset_sizes(n_members: int, sizes=None) -> tuple:
    chosen = DEFAULT_SUBSET_SIZES if sizes is None else tuple(sizes)
    out = tuple(int(k) for k in chosen if 1 <= int(k) <= n_members)
    if not out:
        raise ConfigError(f"no usable subset sizes for {n_members} members")
    return out


def ensemble_curve(members, truth, spec: GridSpec, sizes=None, wavelength_km=None) -> list:
    """RMSE (and optionally mean blur over times) of the leading-k ensemble mean, one row per subset size
    (evaluation.py:134-166).  members: (n, rows, cols) or (n, times, rows, cols), host or device."""
    m = _device(members)
    if m.dim() == 3:
        m = m[:, None]
    if m.dim() != 4 or tuple(m.shape[2:]) != (spec.rows, spec.cols):
        raise DataError(f"members must be (n, times, {spec.rows}, {spec.cols}); got {tuple(m.shape)}")
    t = _time_stack(_device(truth), spec, "truth")
    if tuple(m.shape[1:]) != tuple(t.shape):
        raise DataError(f"member shape {tuple(m.shape[1:])} vs truth {tuple(t.shape)}")
    if m.dtype != t.dtype:
        m, t = m.double(), t.double()
    m = m.contiguous()
    truth_power = None
    rows = []
    for k in subset_sizes(m.shape[0], sizes):
        row = {"size": k, "rmse": _rmse_from(m, k, t, spec)}
        if wavelength_km is not None:
            if truth_power is None:
                truth_power = _zonal_power_dev(t, 1, spec)
            mean_power = _zonal_power_dev(m, k, spec)
            wm, wt = _interp_rows(mean_power, spec, wavelength_km), _interp_rows(truth_power, spec, wavelength_km)
            blurs = [_blur_from_powers(float(wm[i]), float(wt[i])) for i in range(t.shape[0])]
            row["blur"] = float(np.mean(blurs))
        rows.append(row)
    return rows


def plane_scores(pred, truth, spec: GridSpec, wavelength_km: float):
    """Per-plane RMSE and blur of (P, rows, cols) forecast planes against truth planes, all planes in one
    launch per metric (the `evaluate` command's loop of cli.py:244-256, batched).  Returns (rmse[P], blur[P])
    with blur None where unbounded."""
    p, g = _device(pred), _device(truth)
    if p.shape != g.shape or p.dim() != 3 or tuple(p.shape[1:]) != (spec.rows, spec.cols):
        raise DataError(f"plane stacks must match and be (P, {spec.rows}, {spec.cols}); got {tuple(p.shape)} "
                        f"vs {tuple(g.shape)}")
    if p.dtype != g.dtype:
        p, g = p.double(), g.double()
    n = p.shape[0]
    partial = torch.empty((n, spec.rows), dtype=torch.float64, device="cuda")
    check(_lib.lib().wm3_sq_err_rows(_dtype_code(p), ptr(p), 0, 1, ptr(g), ptr(_weights(spec)), n, spec.rows,
                                     spec.cols, ptr(partial), stream_ptr()), "wm3_sq_err_rows")
    rmse = np.sqrt(partial.cpu().numpy().sum(axis=1) / (spec.rows * spec.cols))
    wf = _interp_rows(_zonal_power_dev(p, 1, spec), spec, wavelength_km)
    wt = _interp_rows(_zonal_power_dev(g, 1, spec), spec, wavelength_km)
    blur = []
    for i in range(n):
        b = _blur_from_powers(float(wf[i]), float(wt[i]))
        blur.append(None if not np.isfinite(b) else b)
    return [float(v) for v in rmse], blur


def scorecard(rmse_a: dict, rmse_b: dict) -> dict:
    """Percent RMSE change of a versus b (negative: a better); NaN for a zero baseline (evaluation.py:173-190)."""
    if set(rmse_a) != set(rmse_b):
        raise DataError(f"scorecard key mismatch: {sorted(set(rmse_a) ^ set(rmse_b))}")
    out = {}
    for k in sorted(rmse_a):
        a, b = float(rmse_a[k]), float(rmse_b[k])
        out[k] = float("nan") if b == 0.0 else 100.0 * (a - b) / b
    return out
