"""Device plumbing: torch tensors as HBM buffers, the current stream, host staging.

PyTorch is used only for device memory and streams; every computation goes
through libmgp.so.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def is_tensor(x) -> bool:
    if _torch is None:
        mod = type(x).__module__
        if not mod.startswith("torch"):
            return False
    return isinstance(x, torch().Tensor)


def is_cuda_tensor(x) -> bool:
    return is_tensor(x) and x.is_cuda


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2109_13504_b200 needs a CUDA device (B200); there is no CPU fallback")
    _lib.lib()


def stream_ptr(device=None):
    t = torch()
    s = t.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def ptr(x):
    """Raw pointer of a contiguous torch tensor or numpy array."""
    if is_tensor(x):
        return ctypes.c_void_p(x.data_ptr())
    return x.ctypes.data_as(ctypes.c_void_p)


def wdtype(x) -> int:
    dt = str(x.dtype)
    if dt.endswith("float32"):
        return _lib.MGP_F32
    if dt.endswith("float64"):
        return _lib.MGP_F64
    raise ValueError(f"weights must be float32 or float64, got {x.dtype}")


def as_index_tensor(a, device):
    """int64 contiguous CUDA tensor view/copy of ancestors."""
    t = torch()
    if is_tensor(a):
        return a.to(device=device, dtype=t.int64).contiguous()
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(device)
