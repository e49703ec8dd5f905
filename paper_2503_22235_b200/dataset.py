"""WMD3 dataset container (gridcast/synthdata.py:80-294): reader/writer plus device-side state extraction.

Byte layout (little-endian, synthdata.py:201-206): b"WMD3" | u32 version (1) | 6 x f64 grid (rows, cols,
north_lat, lat_step, lon_step, planet_radius_km) | u8 flags (bit 0: south pole omitted) | 6 x u32 (surface_in,
surface_out, atmos_vars, levels, n_sources, n_times) | n_times x i64 hours | per time: the truth planes (f32),
then every source's planes (f32), channel-major.

`load_dataset` keeps the reference's contract (DataError for bad magic / version / header / truncation /
trailing bytes; bitwise round trips).  It parses the header, validates the payload size up front, and splits
the time-major payload with one strided view per block (no per-time copy loop).

`WeatherDataset.input_state` matches the reference (float64 host fields).  The B200 path adds
`input_state_device`, which copies one sample's float32 planes straight to the GPU in the (C, H, W) /
(A, L, H, W) layout `model.encode` consumes, skipping the float64 widening the reference does on the host.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .config import GridSpec
from .errors import ConfigError, DataError
from .model import WeatherState

MAGIC = b"WMD3"
VERSION = 1
_SOUTH_POLE_OMITTED = 0x01
_HEAD = struct.Struct("<4sI6dB6I")  # magic, version, grid, flags, channel counts

__all__ = ["WeatherDataset", "dump_dataset", "load_dataset", "save_dataset_file", "load_dataset_file", "MAGIC",
           "VERSION"]


@dataclass
class WeatherDataset:
    """Hourly truth planes plus one or more input sources, float32 at rest (synthdata.py:80-140)."""
    grid: GridSpec
    surface_in: int
    surface_out: int
    atmos_vars: int
    levels: int
    times: np.ndarray  # (T,) int64 hours
    truth: np.ndarray  # (T, surface_out + atmos_vars * levels, rows, cols) float32
    sources: tuple     # each (T, surface_in + atmos_vars * levels, rows, cols) float32

    def __post_init__(self):
        t, (h, w) = self.times.size, (self.grid.rows, self.grid.cols)
        if self.times.dtype != np.int64:
            raise DataError("time axis must be int64 hours")
        want_truth = (t, self.surface_out + self.atmos_vars * self.levels, h, w)
        want_src = (t, self.surface_in + self.atmos_vars * self.levels, h, w)
        if self.truth.shape != want_truth or self.truth.dtype != np.float32:
            raise DataError(f"truth block must be float32 {want_truth}")
        if not self.sources:
            raise DataError("dataset needs at least one input source")
        for s in self.sources:
            if s.shape != want_src or s.dtype != np.float32:
                raise DataError(f"source block must be float32 {want_src}")

    @property
    def n_times(self) -> int:
        return int(self.times.size)

    @property
    def n_sources(self) -> int:
        return len(self.sources)

    def index_at(self, hour: int) -> int:
        i = int(np.searchsorted(self.times, hour))
        if i >= self.times.size or self.times[i] != hour:
            raise DataError(f"no sample at hour {hour}")
        return i

    def _split(self, planes: np.ndarray, n_sfc: int):
        h, w = self.grid.rows, self.grid.cols
        return planes[:n_sfc], planes[n_sfc:].reshape(self.atmos_vars, self.levels, h, w)

    def input_state(self, idx: int, source: int = 0) -> WeatherState:
        """Encoder input at one time as float64 host fields (synthdata.py:126-131)."""
        sfc, atm = self._split(self.sources[source][idx].astype(np.float64), self.surface_in)
        return WeatherState(int(self.times[idx]), sfc, atm)

    def input_state_device(self, idx: int, source: int = 0) -> WeatherState:
        """Encoder input at one time as float32 CUDA tensors (no host widening; encode consumes fp32)."""
        import torch
        planes = torch.from_numpy(np.ascontiguousarray(self.sources[source][idx])).to("cuda", non_blocking=False)
        h, w = self.grid.rows, self.grid.cols
        return WeatherState(int(self.times[idx]), planes[:self.surface_in],
                            planes[self.surface_in:].reshape(self.atmos_vars, self.levels, h, w))

    def truth_fields(self, idx: int):
        """Target planes at one time: surface (S, H, W), atmos (A, L, H, W), float64 (synthdata.py:133-138)."""
        return self._split(self.truth[idx].astype(np.float64), self.surface_out)

    def plane_sigmas(self) -> np.ndarray:
        """Per truth plane standard deviation over all times, floored at 1e-6 (synthdata.py:140-144)."""
        flat = self.truth.reshape(self.n_times, self.truth.shape[1], -1).astype(np.float64)
        return np.maximum(flat.std(axis=(0, 2)), 1e-6)


def dump_dataset(ds: WeatherDataset) -> bytes:
    g = ds.grid
    head = _HEAD.pack(MAGIC, VERSION, float(g.rows), float(g.cols), g.north_lat, g.lat_step, g.lon_step,
                      g.planet_radius_km, _SOUTH_POLE_OMITTED if g.south_pole_omitted else 0, ds.surface_in,
                      ds.surface_out, ds.atmos_vars, ds.levels, ds.n_sources, ds.n_times)
    # time-major payload: per time the truth planes then each source's planes
    per_time = [ds.truth.reshape(ds.n_times, -1)] + [s.reshape(ds.n_times, -1) for s in ds.sources]
    body = np.concatenate([a.astype("<f4", copy=False) for a in per_time], axis=1)
    return head + ds.times.astype("<i8").tobytes() + np.ascontiguousarray(body).tobytes()


def load_dataset(blob) -> WeatherDataset:
    buf = memoryview(blob)
    if len(buf) < 4 or bytes(buf[:4]) != MAGIC:
        raise DataError("not a WMD3 dataset (bad magic)")
    if len(buf) < 8:
        raise DataError("dataset file truncated")
    (version,) = struct.unpack_from("<I", buf, 4)
    if version != VERSION:
        raise DataError(f"unsupported WMD3 version {version}")
    if len(buf) < _HEAD.size:
        raise DataError("dataset file truncated")
    (_, _, rows_f, cols_f, north, lat_step, lon_step, radius, flags, s_in, s_out, a_vars, levels, n_src,
     n_t) = _HEAD.unpack_from(buf, 0)
    if rows_f != int(rows_f) or cols_f != int(cols_f):
        raise DataError("non-integer grid dimensions")
    try:
        grid = GridSpec(rows=int(rows_f), cols=int(cols_f), north_lat=north, lat_step=lat_step, lon_step=lon_step,
                        south_pole_omitted=bool(flags & _SOUTH_POLE_OMITTED), planet_radius_km=radius)
    except ConfigError as e:
        raise DataError(f"invalid grid header: {e}") from e
    if s_in < 1 or s_out < s_in or a_vars < 1 or levels < 1 or n_src < 1:
        raise DataError("invalid channel counts in header")
    off = _HEAD.size
    if len(buf) < off + 8 * n_t:
        raise DataError("dataset file truncated")
    times = np.frombuffer(buf, dtype="<i8", count=n_t, offset=off).astype(np.int64)
    off += 8 * n_t
    hw = grid.rows * grid.cols
    n_truth, n_in = s_out + a_vars * levels, s_in + a_vars * levels
    row = n_truth + n_src * n_in  # float32 planes per time
    need = 4 * n_t * row * hw
    if len(buf) - off < need:
        raise DataError("dataset file truncated")
    if len(buf) - off > need:
        raise DataError(f"{len(buf) - off - need} trailing bytes after dataset")
    body = np.frombuffer(buf, dtype="<f4", count=n_t * row * hw, offset=off).reshape(n_t, row, grid.rows,
                                                                                      grid.cols)
    truth = np.ascontiguousarray(body[:, :n_truth], dtype=np.float32)
    sources = tuple(np.ascontiguousarray(body[:, n_truth + j * n_in:n_truth + (j + 1) * n_in], dtype=np.float32)
                    for j in range(n_src))
    return WeatherDataset(grid=grid, surface_in=s_in, surface_out=s_out, atmos_vars=a_vars, levels=levels,
                          times=times, truth=truth, sources=sources)


def save_dataset_file(ds: WeatherDataset, path) -> None:
    with open(path, "wb") as f:
        f.write(dump_dataset(ds))


def load_dataset_file(path) -> WeatherDataset:
    with open(path, "rb") as f:
        return load_dataset(f.read())
