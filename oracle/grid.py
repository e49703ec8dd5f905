"""Oracle restatement of the reference lat-lon geometry (pkg/src/gridcast/grid.py)."""

from __future__ import annotations

import numpy as np


class OracleConfigError(ValueError):
    """Mirror of gridcast.errors.ConfigError (errors.py:4-5) for oracle-side validation."""


def bump_starts(extent: int, window: int) -> np.ndarray:
    """grid.py:96-101 — window start per center index: slide to fit, never shrink."""
    if window > extent:
        raise OracleConfigError(f"window {window} exceeds axis extent {extent}")
    half = (window - 1) // 2
    return np.clip(np.arange(extent) - half, 0, extent - window)


def neighborhood(extents, window) -> np.ndarray:
    """grid.py:107-130 — (T, K) int64 table; bump on depth/rows, wrap on cols, K order (kd, kh, kw)."""
    d, h, w = (int(e) for e in extents)
    wd, wh, ww = (int(e) for e in window)
    if ww > w:
        raise OracleConfigError(f"window {ww} exceeds axis extent {w}")
    d_idx = bump_starts(d, wd)[:, None] + np.arange(wd)[None, :]
    h_idx = bump_starts(h, wh)[:, None] + np.arange(wh)[None, :]
    w_idx = (np.arange(w)[:, None] + np.arange(ww)[None, :] - (ww - 1) // 2) % w
    flat = (d_idx[:, None, None, :, None, None] * (h * w)
            + h_idx[None, :, None, None, :, None] * w
            + w_idx[None, None, :, None, None, :])
    return np.ascontiguousarray(flat.reshape(d * h * w, wd * wh * ww), dtype=np.int64)


def latitudes(rows: int, north_lat: float, lat_step: float) -> np.ndarray:
    """grid.py:66-67."""
    return north_lat - np.arange(rows) * lat_step


def longitudes(cols: int, lon_step: float) -> np.ndarray:
    """grid.py:70-71."""
    return np.arange(cols) * lon_step


def static_fields(rows: int, cols: int, north_lat: float, lat_step: float, lon_step: float) -> np.ndarray:
    """grid.py:143-174 — 7 deterministic surface descriptor channels, (7, rows, cols) float64."""
    lat = np.radians(latitudes(rows, north_lat, lat_step))[:, None]
    lon = np.radians(longitudes(cols, lon_step))[None, :]
    shape = (rows, cols)
    sin_lat = np.broadcast_to(np.sin(lat), shape)
    cs = np.cos(lat) * np.sin(lon)
    cc = np.cos(lat) * np.cos(lon)
    continents = (np.sin(2 * lat + 0.7) * np.cos(3 * lon - 1.1)
                  + 0.5 * np.sin(5 * lon + 2 * lat)
                  + 0.3 * np.cos(lat * 4 - 0.3))
    land = (continents > 0.15).astype(np.float64)
    soil = np.floor(3.0 * (0.5 + 0.5 * np.sin(3 * lat - lon)))
    soil = np.clip(soil, 0, 2) / 2.0 * land
    topo = land * np.maximum(0.0, continents - 0.15) * (1.0 + 0.4 * np.sin(7 * lon) * np.cos(5 * lat))
    rough = land * np.abs(np.sin(9 * lon + 4 * lat)) * 0.5
    out = np.stack([sin_lat, cs, cc,
                    np.broadcast_to(land, shape), np.broadcast_to(soil, shape),
                    np.broadcast_to(topo, shape), np.broadcast_to(rough, shape)]).astype(np.float64)
    return np.ascontiguousarray(out)
