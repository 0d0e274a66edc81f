"""Device plumbing: torch tensors as HBM buffers, the current CUDA stream, and
host<->device movement for callers that hand in numpy arrays (the reference
API is numpy-in/numpy-out; device tensors in give device tensors out).

PyTorch is used only as an allocator/stream provider: all arithmetic on the
solve path runs in libmpkb200.so."""

from __future__ import annotations

import numpy as np

from . import _lib

_TORCH = None


def torch():
    global _TORCH
    if _TORCH is None:
        import torch as _t

        _TORCH = _t
    return _TORCH


def lib():
    return _lib.load(require_device=True)


def stream() -> int:
    return torch().cuda.current_stream().cuda_stream


def device():
    t = torch()
    return t.device("cuda", t.cuda.current_device())


def is_tensor(v) -> bool:
    t = torch()
    return isinstance(v, t.Tensor)


def np_dtype(v) -> np.dtype:
    if is_tensor(v):
        return np.dtype(str(v.dtype).replace("torch.", ""))
    return np.asarray(v).dtype


def shape(v):
    return tuple(v.shape)


def to_device(v, dtype=None):
    """Return a contiguous CUDA tensor view/copy of v (numpy or torch)."""
    t = torch()
    if is_tensor(v):
        out = v if v.is_cuda else v.to(device(), non_blocking=False)
        if dtype is not None and out.dtype != dtype:
            out = out.to(dtype)
        return out.contiguous()
    a = np.ascontiguousarray(v)
    out = t.from_numpy(a).to(device(), non_blocking=False)
    if dtype is not None and out.dtype != dtype:
        out = out.to(dtype)
    return out


def to_host(t_):
    return t_.detach().cpu().numpy()


def like_input(dev_tensor, was_host):
    """Return the result in the caller's kind: numpy for numpy input, a CPU
    tensor for a CPU tensor input, the device tensor otherwise."""
    if was_host is True:
        return to_host(dev_tensor)
    if was_host == "cpu_tensor":
        return dev_tensor.detach().cpu()
    return dev_tensor


def host_kind(v):
    """True (numpy), 'cpu_tensor', or False (CUDA tensor)."""
    if not is_tensor(v):
        return True
    return False if v.is_cuda else "cpu_tensor"


def empty(n, torch_dtype):
    return torch().empty(int(n), dtype=torch_dtype, device=device())


def zeros(n, torch_dtype):
    return torch().zeros(int(n), dtype=torch_dtype, device=device())


def ptr(t_) -> int:
    return int(t_.data_ptr()) if t_ is not None else 0


def sync():
    torch().cuda.current_stream().synchronize()


class ReduceWorkspace:
    """Scratch for the deterministic grid reductions (ticket counters must start
    at zero; every kernel resets its counter on exit)."""

    _cache: dict = {}

    def __init__(self):
        nbytes = int(lib().mpk_reduce_ws_bytes(0, 64))
        self.buf = torch().zeros(nbytes, dtype=torch().uint8, device=device())

    @property
    def ptr(self) -> int:
        return int(self.buf.data_ptr())

    @classmethod
    def shared(cls) -> "ReduceWorkspace":
        key = torch().cuda.current_device()
        ws = cls._cache.get(key)
        if ws is None:
            ws = cls._cache[key] = ReduceWorkspace()
        return ws


def ld_for(n: int) -> int:
    """Leading dimension of a column-major basis: n rounded up to 64 elements,
    so every column starts on a 256/512-byte boundary."""
    return max(64, (int(n) + 63) // 64 * 64)
