"""Device plumbing: tensors, streams, workspaces, host<->device conversion.

PyTorch is used only for device memory, streams and (optionally) CUDA
graphs; every arithmetic operation on the hot path is a liblsb200 kernel.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _abi
from .errors import DimensionError

F64 = torch.float64


def require_cuda():
    if not torch.cuda.is_available():
        raise _abi.LsbUnavailable("no CUDA device: liblsb200 has no CPU fallback")
    _abi.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def round_up(x, a):
    return (x + a - 1) // a * a


def is_host(x):
    """True for numpy / python / CPU-tensor inputs (results go back to host)."""
    if isinstance(x, torch.Tensor):
        return not x.is_cuda
    return True


def to_device_vector(x, n=None, copy=False):
    """Contiguous, 16-byte aligned float64 CUDA vector (no copy when possible)."""
    dev = require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=F64)
    else:
        a = np.ascontiguousarray(x, dtype=np.float64)
        t = h2d(a, dev) if a.ndim == 1 and a.size >= _STAGE_MIN else torch.as_tensor(a, device=dev)
    if t.dim() != 1:
        raise DimensionError(f"expected a vector, got shape {tuple(t.shape)}")
    if n is not None and t.shape[0] != n:
        raise DimensionError(f"expected length {n}, got {t.shape[0]}")
    if copy or not t.is_contiguous() or t.data_ptr() % 16:
        t = _aligned_copy(t)
    return t


def _aligned_copy(t):
    out = torch.empty(t.shape[0], dtype=F64, device=t.device)  # fresh: 512-byte aligned
    out.copy_(t)
    return out


def colmajor(X):
    """(n, p) block as (tensor, ptr, ld) with unit row stride, even ld, 16-byte
    aligned base (KrylovBasis views satisfy this without copies)."""
    dev = require_cuda()
    if not isinstance(X, torch.Tensor):
        X = torch.as_tensor(np.asarray(X, dtype=np.float64))
    X = X.to(device=dev, dtype=F64)
    if X.dim() != 2:
        raise ValueError("basis must be a 2-d column block")
    n, p = X.shape
    ok = (p <= 1 or X.stride(1) % 2 == 0) and (X.stride(0) == 1 or n <= 1) and X.data_ptr() % 16 == 0
    if p == 0:
        return X, None, max(2, round_up(n, 2))
    if ok:
        ld = X.stride(1) if p > 1 else round_up(max(n, 2), 2)
        return X, C.c_void_p(X.data_ptr()), ld
    ld = round_up(max(n, 2), 32)
    store = torch.zeros((p, ld), dtype=F64, device=dev)
    store[:, :n].copy_(X.t())
    view = store[:, :n].t()
    return view, C.c_void_p(store.data_ptr()), ld


def out_like(t, like_host):
    """Return a device result in the caller's world (numpy in -> numpy out)."""
    if like_host:
        if t.dim() == 1 and t.numel() >= _STAGE_MIN:
            return d2h(t)
        return t.detach().cpu().numpy()
    return t


# Large host<->device vector copies go through one cached pinned staging
# buffer: pageable cudaMemcpy of a 134 MB vector runs at ~2 GB/s on the
# B200 host, pinned DMA at ~50 GB/s plus a ~40 GB/s host memcpy.
_STAGE_MIN = 1 << 16
_stage = threading.local()   # one staging buffer per host thread (in-process ranks)


def _staging(n):
    buf = getattr(_stage, "buf", None)
    if buf is None or buf.numel() < n:
        buf = _stage.buf = torch.empty(max(n, 1 << 20), dtype=F64).pin_memory()
    return buf[:n]


def h2d(a, dev):
    st = _staging(a.size)
    st.copy_(torch.from_numpy(a))               # multi-threaded host copy
    out = torch.empty(a.size, dtype=F64, device=dev)
    out.copy_(st, non_blocking=True)
    torch.cuda.current_stream().synchronize()   # staging buffer is reused
    return out


def d2h(t):
    st = _staging(t.numel())
    st.copy_(t.detach(), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    out = torch.empty(t.numel(), dtype=F64)     # fresh result owned by numpy
    out.copy_(st)                               # multi-threaded host copy
    return out.numpy()


class Workspace:
    """Reduction scratch (per-CTA partials + self-resetting counter)."""

    def __init__(self, pmax=256, device=None):
        device = device or require_cuda()
        lib = _abi.load()
        self.partial = torch.zeros(int(lib.lsb_partial_len(int(pmax))), dtype=F64, device=device)
        self.counter = torch.zeros(8, dtype=torch.int32, device=device)
        self.c = _abi.Workspace(self.partial.data_ptr(), self.counter.data_ptr(), 0, 0)

    def ref(self):
        return C.byref(self.c)


_ws_cache = {}


def default_workspace():
    dev = require_cuda()
    key = (dev.index, torch.cuda.current_stream().cuda_stream)
    ws = _ws_cache.get(key)
    if ws is None:
        ws = _ws_cache[key] = Workspace(256, dev)
    return ws
