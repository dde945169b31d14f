"""Host logic of the engine cache (gmres._cached_engine / _BasisSnapshot) on
CPU tensors: a live history whose lazy basis still reads the cached engine
is detached onto a device copy before the engine is reused, bases above the
size limit get a fresh engine instead, and a snapshot answers basis() /
hessenberg() exactly as the engine would have."""

import types
import weakref

import numpy as np
import pytest
import torch

from paper_1809_05805_b200 import gmres as gm


class _Eng(types.SimpleNamespace):
    basis = gm.Engine.basis
    hessenberg = gm.Engine.hessenberg


def _engine(n=37, cap=6, off=2):
    g = torch.Generator().manual_seed(3)
    V = torch.randn((cap, off + n + 5), generator=g, dtype=torch.float64)
    R = torch.randn((cap, cap), generator=g, dtype=torch.float64)
    return _Eng(n=n, off=off, Vstore=V, R=R)


class _A:        # weak-referenceable operator stand-in
    pass


def _entry(eng, A, hist):
    return (eng, weakref.ref(A), weakref.ref(hist))


def test_snapshot_detaches_live_history():
    gm.clear_engine_cache()
    eng, A, h = _engine(), _A(), gm.ConvergenceHistory()
    k, ncols = 4, 5
    h._stash = (eng, k, ncols)
    want_b, want_h = eng.basis(k, ncols), eng.hessenberg(k)
    gm._ENGINE_CACHE["key"] = _entry(eng, A, h)
    assert gm._cached_engine("key", A) is eng
    assert isinstance(h._stash[0], gm._BasisSnapshot)
    eng.Vstore.zero_()             # the reused engine overwrites its storage
    eng.R.zero_()
    assert np.array_equal(h.basis, want_b)
    assert np.array_equal(h.hessenberg, want_h)
    gm.clear_engine_cache()


def test_released_or_read_history_needs_no_snapshot():
    eng, A, h = _engine(), _A(), gm.ConvergenceHistory()
    h._stash = (eng, 3, 4)
    h.basis                         # materialised: nothing left to protect
    gm._ENGINE_CACHE["key"] = _entry(eng, A, h)
    assert gm._cached_engine("key", A) is eng and h._stash[0] is eng
    h.release()
    assert gm._cached_engine("key", A) is eng and h._stash is None
    gm.clear_engine_cache()


def test_large_basis_gets_a_fresh_engine(monkeypatch):
    monkeypatch.setattr(gm, "_SNAPSHOT_MAX_BYTES", 64)
    eng, A, h = _engine(), _A(), gm.ConvergenceHistory()
    h._stash = (eng, 4, 5)
    gm._ENGINE_CACHE["key"] = _entry(eng, A, h)
    assert gm._cached_engine("key", A) is None
    assert h._stash[0] is eng       # untouched: the old engine stays with it
    gm.clear_engine_cache()


def test_other_operator_object_is_a_miss():
    eng, A, h = _engine(), _A(), gm.ConvergenceHistory()
    gm._ENGINE_CACHE["key"] = _entry(eng, A, h)
    assert gm._cached_engine("key", _A()) is None
    assert gm._cached_engine("nokey", A) is None
    gm.clear_engine_cache()
