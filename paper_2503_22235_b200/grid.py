"""Lat-lon geometry of the drop-in API (gridcast/grid.py): grid specs, windows, static fields.

`neighborhood` is the bit-exact export of the window arithmetic the kernels use (wm3_neighbor_table,
computed on the GPU); `bump_starts` is the host-side helper used for band/halo sizing.  `static_fields` builds
the 7 deterministic surface descriptor channels the encoder appends to the surface input (grid.py:143-174);
it runs once per grid on the host and is then resident on the device.
"""

from __future__ import annotations

import math

import numpy as np

from .config import N_STATIC_FIELDS, GridSpec, desk_grid, quarter_degree_grid  # noqa: F401
from .errors import ConfigError

__all__ = ["GridSpec", "quarter_degree_grid", "desk_grid", "latitudes", "longitudes", "latitude_weights",
           "row_circumference_km", "bump_starts", "neighborhood", "static_fields", "N_STATIC_FIELDS"]


def latitudes(spec: GridSpec) -> np.ndarray:
    return spec.north_lat - spec.lat_step * np.arange(spec.rows)


def longitudes(spec: GridSpec) -> np.ndarray:
    return spec.lon_step * np.arange(spec.cols)


def latitude_weights(spec: GridSpec) -> np.ndarray:
    w = np.cos(np.radians(latitudes(spec)))
    if np.any(w <= 0):
        raise ConfigError("nonpositive latitude weight; grid rows reach past a pole")
    return w


def row_circumference_km(spec: GridSpec) -> np.ndarray:
    return 2.0 * math.pi * spec.planet_radius_km * latitude_weights(spec)


def bump_starts(extent: int, window: int) -> np.ndarray:
    """Window start per centre index: clip(i - (w-1)//2, 0, E - w) (grid.py:96-101)."""
    if window > extent:
        raise ConfigError(f"window {window} exceeds axis extent {extent}")
    return np.minimum(np.maximum(np.arange(extent) - (window - 1) // 2, 0), extent - window)


def neighborhood(extents, window) -> np.ndarray:
    """(T, K) int64 neighbor table exported from the device window arithmetic (grid.py:107-130)."""
    d, h, w = (int(e) for e in extents)
    wd, wh, ww = (int(e) for e in window)
    for win, ext in ((ww, w), (wd, d), (wh, h)):
        if win > ext:
            raise ConfigError(f"window {win} exceeds axis extent {ext}")
    from . import ops
    return ops.neighbor_table((d, h, w), (wd, wh, ww)).cpu().numpy()


_STATICS: dict = {}


def static_fields(spec: GridSpec) -> np.ndarray:
    """(7, rows, cols) float64: sin(lat), cos(lat)sin(lon), cos(lat)cos(lon), land mask, soil class, topography,
    roughness — smooth harmonics of position (grid.py:143-174)."""
    hit = _STATICS.get(spec)
    if hit is not None:
        return hit
    lat = np.radians(latitudes(spec))[:, None]
    lon = np.radians(longitudes(spec))[None, :]
    full = (spec.rows, spec.cols)
    relief = np.sin(2 * lat + 0.7) * np.cos(3 * lon - 1.1) + 0.5 * np.sin(5 * lon + 2 * lat) \
        + 0.3 * np.cos(lat * 4 - 0.3)
    land = (relief > 0.15).astype(np.float64)
    soil = np.clip(np.floor(3.0 * (0.5 + 0.5 * np.sin(3 * lat - lon))), 0, 2) / 2.0 * land
    topo = land * np.maximum(0.0, relief - 0.15) * (1.0 + 0.4 * np.sin(7 * lon) * np.cos(5 * lat))
    rough = land * np.abs(np.sin(9 * lon + 4 * lat)) * 0.5
    chans = [np.sin(lat), np.cos(lat) * np.sin(lon), np.cos(lat) * np.cos(lon), land, soil, topo, rough]
    out = np.ascontiguousarray(np.stack([np.broadcast_to(c, full) for c in chans]).astype(np.float64))
    out.setflags(write=False)
    _STATICS[spec] = out
    return out
