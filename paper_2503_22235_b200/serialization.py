"""LMTW parameter container (gridcast/serialization.py), with a direct-to-device loader.

Byte layout (little-endian), as the reference writes it (serialization.py:3-16):
    b"LMTW" | u32 version (1) | u32 count | per entry, names sorted: u32 name_len | utf-8 name | u32 rank |
    rank x u64 extents | prod(extents) x f64 (C order)

`load_params` / `dump_params` / `*_file` keep the reference's contract: bitwise round trips, `ContainerError`
(a ValueError) for a bad magic, an unknown version, truncation or trailing bytes.

The B200 addition is `load_params_device`: the file is memory-mapped, only the small header index is parsed on
the host, and each tensor's float64 payload is copied host->device straight out of the mapping (no
intermediate numpy copy) and narrowed to fp32 on the GPU.  At full scale (452 tensors, 3.06 GB) this replaces
a 3 GB host copy plus per-tensor conversion with one streaming pass.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"LMTW"
VERSION = 1

__all__ = ["ContainerError", "dump_params", "load_params", "save_params_file", "load_params_file",
           "index_params", "load_params_device", "MAGIC", "VERSION"]


class ContainerError(ValueError):
    """Malformed or truncated parameter container (serialization.py:26-27)."""


def _as_f64(v) -> np.ndarray:
    from .tensor import host_array
    a = host_array(v)
    # np.array keeps rank 0 as rank 0 (np.ascontiguousarray would promote it to rank 1)
    return np.array(a, dtype=np.float64, order="C", copy=None)


def dump_params(params: dict) -> bytes:
    """Serialise name -> array (anything with .values, numpy, or torch) to LMTW bytes, names sorted."""
    chunks = [MAGIC + struct.pack("<II", VERSION, len(params))]
    for name in sorted(params):
        arr = _as_f64(params[name])
        raw = name.encode("utf-8")
        head = struct.pack("<I", len(raw)) + raw + struct.pack("<I", arr.ndim)
        if arr.ndim:
            head += struct.pack(f"<{arr.ndim}Q", *arr.shape)
        chunks.append(head)
        chunks.append(arr.astype("<f8", copy=False).tobytes())
    return b"".join(chunks)


def index_params(buf) -> list[tuple[str, tuple[int, ...], int]]:
    """Parse the container index: [(name, shape, byte offset of the f64 payload)], validating the whole
    layout (magic, version, every length against the buffer, no trailing bytes)."""
    view = memoryview(buf)
    size = len(view)

    def take(off: int, n: int, what: str) -> int:
        if n < 0 or off + n > size:
            raise ContainerError(f"truncated container: {what} needs {n} bytes at offset {off}, have {size - off}")
        return off + n

    end = take(0, 12, "header")
    if bytes(view[:4]) != MAGIC:
        raise ContainerError(f"bad magic {bytes(view[:4])!r}, expected {MAGIC!r}")
    version, count = struct.unpack_from("<II", view, 4)
    if version != VERSION:
        raise ContainerError(f"unsupported container version {version}")
    entries = []
    off = end
    for _ in range(count):
        nxt = take(off, 4, "name length")
        (nlen,) = struct.unpack_from("<I", view, off)
        off = take(nxt, nlen, "name")
        name = bytes(view[nxt:off]).decode("utf-8")
        nxt = take(off, 4, "rank")
        (rank,) = struct.unpack_from("<I", view, off)
        off = take(nxt, 8 * rank, f"extents of {name!r}")
        shape = tuple(int(e) for e in struct.unpack_from(f"<{rank}Q", view, nxt)) if rank else ()
        count_vals = int(np.prod(shape, dtype=np.int64)) if shape else 1
        payload = off
        off = take(off, 8 * count_vals, f"values of {name!r}")
        entries.append((name, shape, payload))
    if off != size:
        raise ContainerError(f"{size - off} trailing bytes after last parameter")
    return entries


def load_params(buf) -> dict[str, np.ndarray]:
    """LMTW bytes -> name -> float64 array (fresh, writable copies, as the reference returns)."""
    out = {}
    for name, shape, off in index_params(buf):
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        out[name] = np.frombuffer(buf, dtype="<f8", count=n, offset=off).reshape(shape).astype(np.float64)
    return out


def save_params_file(path, params: dict) -> None:
    with open(path, "wb") as f:
        f.write(dump_params(params))


def load_params_file(path) -> dict[str, np.ndarray]:
    with open(path, "rb") as f:
        return load_params(f.read())


def load_params_device(path, dtype=None, device: str = "cuda") -> dict:
    """Stream an LMTW file to the device (float64 payload -> `dtype`, default fp32): name -> torch tensor.

    The file is read once with readinto() into one page-locked host buffer (no intermediate Python bytes or
    per-tensor numpy copies), the header index is parsed from it, every payload is copied host -> device
    asynchronously from that buffer, and narrowed to `dtype` on the GPU."""
    import torch
    dtype = torch.float32 if dtype is None else dtype
    with open(path, "rb") as f:
        size = f.seek(0, 2)
        if size == 0:
            raise ContainerError("truncated container: empty file")
        f.seek(0)
        host = torch.empty(size, dtype=torch.uint8, pin_memory=(device != "cpu"))
        view = memoryview(host.numpy())
        got = 0
        while got < size:
            k = f.readinto(view[got:])
            if not k:
                raise ContainerError("truncated container: short read")
            got += k
    entries = index_params(view)
    out = {}
    for name, shape, off in entries:
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        raw = host[off:off + 8 * n]  # payloads are not 8-byte aligned in the file: move bytes, view on arrival
        dev = torch.empty(8 * n, dtype=torch.uint8, device=device)
        dev.copy_(raw, non_blocking=True)
        out[name] = dev.view(torch.float64).to(dtype).view(shape)
    if device != "cpu":
        torch.cuda.synchronize()
    return out
