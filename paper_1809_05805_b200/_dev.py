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


_preloaded = set()


def require_cuda():
    if not torch.cuda.is_available():
        raise _abi.LsbUnavailable("no CUDA device: liblsb200 has no CPU fallback")
    lib = _abi.load()
    dev = torch.cuda.current_device()
    if dev not in _preloaded:
        # every liblsb200 kernel loaded up front (lsb_preload): a lazy first
        # launch would wait for the device to idle (deadlock-prone while a
        # peer exchange spins) and would land inside timed regions
        torch.cuda.init()
        torch.zeros(1, device=torch.device("cuda", dev))   # context exists
        if lib.lsb_preload() < 0:
            import warnings
            warnings.warn("lsb_preload: " + lib.lsb_last_error().decode(errors="replace"))
        _preloaded.add(dev)
    return torch.device("cuda", dev)


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


def out_like(t, like_host, host_out=None):
    """Return a device result in the caller's world (numpy in -> numpy out).
    Large vectors land in page-locked memory by one DMA and are handed out
    as numpy arrays over it (torch's pinned caching allocator: once the
    caller drops the array its buffer serves the next result, so steady-state
    solves neither allocate nor stage through a host memcpy -- C2: 6.4 ms of
    staged D2H -> one ~2.7 ms DMA).  host_out: a HostBuffer for the staged
    fallback (page-locking a caller's buffer instead measured slower:
    cudaHostUnregister of 134 MB costs more than the copy it saves)."""
    if like_host:
        if t.dim() == 1 and t.numel() >= _STAGE_MIN:
            if _PINNED_RESULTS:
                try:
                    out = torch.empty(t.numel(), dtype=F64, pin_memory=True)
                except RuntimeError:
                    out = None
                if out is not None:
                    out.copy_(t.detach(), non_blocking=True)
                    torch.cuda.current_stream().synchronize()
                    return out.numpy()
            return d2h(t, host_out.get() if host_out is not None else None)
        return t.detach().cpu().numpy()
    return t


import os as _os
_PINNED_RESULTS = _os.environ.get("LSB_PINNED_RESULTS", "1") != "0"


class HostBuffer:
    """A fresh n-double host result buffer whose pages are faulted in by a
    background thread while the device works: the first touch of 134 MB of
    fresh pageable memory (kernel zero-fill, ~20 GB/s) would otherwise sit
    inside the device->host copy of the solution."""

    def __init__(self, n):
        self.n = n
        self.buf = None
        self.th = threading.Thread(target=self._fill, daemon=True)
        self.th.start()

    def _fill(self):
        b = torch.empty(self.n, dtype=F64)
        b.zero_()                     # releases the GIL; faults every page in
        self.buf = b

    def get(self):
        self.th.join()
        return self.buf


# Large host<->device vector copies go through cached pinned staging
# buffers: pageable cudaMemcpy of a 134 MB vector runs at ~2 GB/s on the
# B200 host, pinned DMA at ~50 GB/s plus a ~40 GB/s host memcpy.  The copy is
# chunked over two staging buffers so the host memcpy of one chunk overlaps
# the DMA of the other.
_STAGE_MIN = 1 << 16
_CHUNK = 1 << 22            # 32 MB per staging chunk
_stage = threading.local()   # staging buffers per host thread (in-process ranks)


def _staging():
    st = getattr(_stage, "bufs", None)
    if st is None:
        st = _stage.bufs = [(torch.empty(_CHUNK, dtype=F64).pin_memory(), torch.cuda.Event())
                            for _ in range(2)]
        for _, ev in st:
            ev.record()
    return st


def h2d(a, dev):
    n = a.size
    src = torch.from_numpy(a)
    out = torch.empty(n, dtype=F64, device=dev)
    if src.is_pinned():
        # the caller's array already sits in page-locked memory (e.g. a
        # numpy view of a pinned torch tensor): one DMA, no staging memcpy.
        # Stream-ordered before every kernel that reads it; the solve
        # synchronises before returning, so `a` is free again by then.
        out.copy_(src, non_blocking=True)
        return out
    bufs = _staging()
    for i, lo in enumerate(range(0, n, _CHUNK)):
        hi = min(n, lo + _CHUNK)
        buf, ev = bufs[i % 2]
        ev.synchronize()                         # DMA out of this buffer finished
        buf[:hi - lo].copy_(src[lo:hi])          # multi-threaded host copy
        out[lo:hi].copy_(buf[:hi - lo], non_blocking=True)
        ev.record()
    torch.cuda.current_stream().synchronize()   # staging buffers are reused
    return out


def d2h(t, out=None):
    t = t.detach()
    n = t.numel()
    if out is None or out.numel() != n:
        out = torch.empty(n, dtype=F64)          # fresh result owned by numpy
    bufs = _staging()
    spans = [(lo, min(n, lo + _CHUNK)) for lo in range(0, n, _CHUNK)]

    def issue(i):
        lo, hi = spans[i]
        buf, ev = bufs[i % 2]
        buf[:hi - lo].copy_(t[lo:hi], non_blocking=True)
        ev.record()

    issue(0)
    for i, (lo, hi) in enumerate(spans):
        if i + 1 < len(spans):
            issue(i + 1)                         # DMA of the next chunk overlaps ...
        buf, ev = bufs[i % 2]
        ev.synchronize()
        out[lo:hi].copy_(buf[:hi - lo])          # ... the host copy of this one
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
