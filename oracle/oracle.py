"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU oracle (fps_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline; the product package never imports it.

Besides the C restatement of ``run_kernel`` (fps_core.py:110-175) this module
restates the thin host layers above it so that tests can compare whole
pipelines:

* ``fps_prune``          pkg/src/flashfps/fps_prune.py:68-111 (slice fill only)
* ``kernel_budget`` / ``candidate_count``  fps_prune.py:45-51 (IEEE double floor)
* ``hierarchical``       pkg/src/flashfps/fps_cache.py:204-240 (cache on/off)

Parity pinning: tests/test_oracle.py checks this oracle against the golden
vectors in tests/golden/ produced by the unmodified reference
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libffps_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH)
                < os.path.getmtime(os.path.join(_HERE, "fps_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        for suf in ("f32", "f64"):
            f = getattr(L, f"ffps_oracle_run_kernel_{suf}")
            f.restype = i64
            f.argtypes = [vp, i64, i64, i64, vp, vp, vp]
        L.ffps_oracle_fill_slice.restype = ctypes.c_int
        L.ffps_oracle_fill_slice.argtypes = [vp, i64, i64, i64, vp]
        L.ffps_oracle_run_kernel_batch.restype = ctypes.c_int
        L.ffps_oracle_run_kernel_batch.argtypes = [
            ctypes.c_int, vp, i64, i64, i64, i64, vp, vp, i64, vp, vp, i64,
            ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def run_kernel(points, m: int, seed_pos: int, index_map=None):
    """(order int64[m], sel_d2 T[m], evals) — positions mapped through
    index_map when given (fps_cache.py:195-197). dtype follows ``points``."""
    pts = np.ascontiguousarray(points)
    if pts.dtype not in (np.float32, np.float64):
        pts = pts.astype(np.float64)
    n = pts.shape[0] if index_map is None else int(np.asarray(index_map).shape[0])
    imap = None if index_map is None else np.ascontiguousarray(index_map, dtype=np.int64)
    order = np.empty(m, dtype=np.int64)
    sel = np.empty(m, dtype=pts.dtype)
    fn = lib().ffps_oracle_run_kernel_f32 if pts.dtype == np.float32 \
        else lib().ffps_oracle_run_kernel_f64
    evals = fn(_ptr(pts), n, m, seed_pos, _ptr(imap), _ptr(order), _ptr(sel))
    if evals < 0:
        raise MemoryError("oracle allocation failed")
    return order, sel, int(evals)


def run_kernel_batch(xyz, m: int, seeds, n: int | None = None, index_map=None,
                     threads: int | None = None):
    """xyz (B, N, 3) f32/f64; the kernel runs on the first n points of each
    cloud (candidate prefix) or on xyz[b][index_map[b]]."""
    xyz = np.ascontiguousarray(xyz)
    B, N = xyz.shape[0], xyz.shape[1]
    if index_map is not None:
        index_map = np.ascontiguousarray(index_map, dtype=np.int64)
        n = index_map.shape[1]
    elif n is None:
        n = N
    seeds = np.ascontiguousarray(np.broadcast_to(np.asarray(seeds, dtype=np.int64), (B,)))
    order = np.empty((B, m), dtype=np.int64)
    sel = np.empty((B, m), dtype=xyz.dtype)
    threads = threads or os.cpu_count() or 1
    lib().ffps_oracle_run_kernel_batch(
        0 if xyz.dtype == np.float32 else 1, _ptr(xyz), B, N, n, m, _ptr(seeds),
        _ptr(index_map), 0 if index_map is None else index_map.shape[1],
        _ptr(order), _ptr(sel), m, int(threads))
    return order, sel


def fill_slice(order_k, n: int, fill_n: int):
    order_k = np.ascontiguousarray(order_k, dtype=np.int64)
    out = np.empty(fill_n, dtype=np.int64)
    rc = lib().ffps_oracle_fill_slice(_ptr(order_k), order_k.shape[0], n, fill_n, _ptr(out))
    if rc != 0:
        raise RuntimeError(f"oracle fill failed rc={rc}")
    return out


def kernel_budget(p: float, m1: int) -> int:
    return max(1, math.floor((1.0 - p) * m1))          # fps_prune.py:45-47


def candidate_count(p: float, n: int, m1: int) -> int:
    return max(kernel_budget(p, m1), math.floor((1.0 - p) * n))   # fps_prune.py:49-51


def fps_prune(points, m1: int, p: float, seed: int = 0):
    """Slice-fill FPS-Prune (fps_prune.py:68-111): (indices, sel_d2, k, c)."""
    n = points.shape[0]
    k = kernel_budget(p, m1)
    c = min(candidate_count(p, n, m1), n)
    order, sel, _ = run_kernel(np.ascontiguousarray(points[:c]), k, seed)
    fill_n = m1 - k
    if fill_n > 0:
        fill = fill_slice(order, n, fill_n)
        order = np.concatenate([order, fill])
        sel = np.concatenate([sel, np.zeros(fill_n, dtype=sel.dtype)])
    return order, sel, k, c


def hierarchical(points, budgets, p: float, seed: int = 0, cache_enabled=True):
    """fps_cache.py:204-240 with slice fill: list of (indices, sel_d2)."""
    idx, sel, k, _ = fps_prune(points, budgets[0], p, seed)
    layers = [(idx, sel)]
    for m in budgets[1:]:
        if cache_enabled:
            layers.append((layers[0][0][:m].copy(), layers[0][1][:m].copy()))
        else:
            prev = layers[-1][0]
            o, s, _ = run_kernel(points, m, 0, index_map=prev)
            layers.append((o, s))
    return layers
