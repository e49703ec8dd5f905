"""Minimal `Tensor` with the read surface of gridcast.autodiff.Tensor (autodiff.py:182-271).

Callers of the reference read `.values` (float64, C-contiguous numpy; cli.py:218-219, model.py:173-175),
`.shape`, `.size`, `.nbytes`.  Here a Tensor is backed either by a host array (parameters, user inputs)
or by a device torch tensor (latents, decoded fields); `.values` copies device data to the host once,
as float64, on first access.  `.device` exposes the torch tensor without a copy.
"""

from __future__ import annotations

import zlib

import numpy as np
import torch


class Tensor:
    __slots__ = ("_host", "_dev", "requires_grad", "__weakref__")

    def __init__(self, values=None, requires_grad: bool = False, device: torch.Tensor | None = None):
        if (values is None) == (device is None):
            raise ValueError("Tensor needs exactly one of host values or a device tensor")
        self._host = None if values is None else np.ascontiguousarray(np.asarray(values, dtype=np.float64))
        self._dev = device
        self.requires_grad = bool(requires_grad)

    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            self._host = device_to_host_f64(self._dev.detach())
        return self._host

    @values.setter
    def values(self, v) -> None:
        self._host = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
        self._dev = None

    @property
    def device(self) -> torch.Tensor | None:
        return self._dev

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self._dev.shape) if self._host is None else self._host.shape

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))

    @property
    def nbytes(self) -> int:
        return self.size * 8

    def __repr__(self) -> str:
        where = "host" if self._host is not None else "cuda"
        return f"Tensor(shape={self.shape}, {where})"


def device_to_host_f64(t: torch.Tensor) -> np.ndarray:
    """float64, C-contiguous numpy copy of a tensor.  Device tensors are widened on the device and downloaded
    into page-locked memory (torch's caching host allocator reuses the blocks): a pageable download of the
    0.66 GB full-scale latent ran at ~2 GB/s.  The array keeps its page-locked buffer alive."""
    if t.device.type != "cuda":
        return np.ascontiguousarray(t.to(torch.float64).numpy())
    h = torch.empty(tuple(t.shape), dtype=torch.float64, pin_memory=True)
    h.copy_(t.to(torch.float64))
    return h.numpy()


def payload(x):
    """The array object behind x: a torch tensor as is (torch.Tensor.values is a sparse-tensor method, not
    data), else x.values for our / the reference's Tensor, else x itself."""
    if isinstance(x, torch.Tensor):
        return x
    return getattr(x, "values", x)


def host_array(x, dtype=None) -> np.ndarray:
    """numpy view / copy of x (torch CPU or CUDA tensor, Tensor with .values, or array-like)."""
    v = payload(x)
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().numpy()
    return np.asarray(v, dtype=dtype)


def host_values(t) -> np.ndarray:
    """float64 numpy view of a parameter given as our Tensor, a reference Tensor (.values), a torch tensor
    (e.g. from serialization.load_params_device) or an array."""
    return host_array(t, np.float64)


# at most this many elements of a host parameter array are hashed per content check
TAG_SAMPLES = 256


def content_tag(x) -> tuple:
    """Cheap identity-and-content fingerprint of a parameter, for the device weight caches.

    The reference updates parameters in place (training.py:144, `p.values -= ...`; an `np.copyto` checkpoint
    reload does the same), which keeps the array's identity.  The tag therefore combines the identity with a
    content sample: for a host array, a CRC of up to TAG_SAMPLES evenly strided elements (every element of a
    vector of that size or less); for a torch tensor, torch's in-place version counter and its storage
    address.  A dense update (any optimizer step, any reload) changes the sample; a sparse in-place write to
    a large array may not — call runtime.invalidate_params() after one."""
    v = payload(x)
    if isinstance(v, torch.Tensor):
        return (id(v), v._version, v.data_ptr())
    a = np.asarray(v)
    flat = a.reshape(-1)
    step = max(1, flat.size // TAG_SAMPLES)
    sample = np.ascontiguousarray(flat[::step])
    return (id(v), flat.size, zlib.crc32(sample.view(np.uint8)))
