"""ctypes binding of the C ABI in include/flashfps_b200.h.

The library (``_lib/libflashfps_b200.so``, built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2604_17720_b200/csrc``) is the
only compute path: if it is missing, or no CUDA device is usable, every call
raises KernelError — there is no CPU fallback.  ctypes.CDLL releases the GIL
for the duration of each foreign call.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import KernelError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                        "libflashfps_b200.so")
# A/B builds of the same sources (tools/build_variant.sh) are loaded through
# FFPS_LIB_VARIANT=<name> -> _lib/variants/libflashfps_b200_<name>.so
if os.environ.get("FFPS_LIB_VARIANT"):
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), "variants",
                            f"libflashfps_b200_{os.environ['FFPS_LIB_VARIANT']}.so")

F32, F64 = 0, 1
F32_F64 = 2   # float coordinates, binary64 arithmetic (FFPS_F32_F64)
STATS_WORDS = 4
ALGO = {"auto": 0, "stream": 1, "bucket": 2, "grid": 4,
        # K1g with a fixed number of CTAs per cloud (FFPS_ALGO_GRID_CL(c))
        "grid@1": 4 | 1 << 8, "grid@2": 4 | 2 << 8, "grid@4": 4 | 4 << 8, "small": 5}
_STATUS = {-1: "EINVAL", -2: "EUNSUPPORTED", -3: "ECUDA"}

_lock = threading.Lock()
_lib = None

# (symbol, restype, argtypes) — must match include/flashfps_b200.h
_i64, _vp, _int = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
SIGNATURES = {
    "ffps_run_kernel": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp,
                               _vp, _i64, _vp]),
    "ffps_run_kernel_ex": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp,
                                  _vp, _i64, _vp, _int]),
    "ffps_run_kernel_stats": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp,
                                     _vp, _i64, _vp, _int, _vp]),
    "ffps_trim_scratch": (_int, []),
    "ffps_hierarchical_sample": (_int, [_int, _vp, _i64, _i64, _i64, ctypes.POINTER(_i64), _int,
                                        _i64, _i64, _int, ctypes.POINTER(ctypes.c_uint64), _int,
                                        _vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "ffps_fill_slice": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _i64, _vp]),
    "ffps_fill_random": (_int, [_int, _vp, _vp, _i64, _i64, _i64, _i64, _i64, ctypes.c_uint64,
                                ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _vp]),
    "ffps_coverage": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp]),
    "ffps_plan": (_int, [_int, _i64, _i64, ctypes.POINTER(_i64)]),
    "ffps_bucket_plan": (_int, [_int, _i64, ctypes.POINTER(_i64)]),
    "ffps_auto_schedule": (_int, [_i64, _i64]),
    "ffps_auto_schedule_ex": (_int, [_i64, _i64, _int]),
    "ffps_grid_plan": (_int, [_int, _i64, _i64, _int, ctypes.POINTER(_i64)]),
    "ffps_h2d_prefix": (_int, [_vp, _vp, _i64, _i64, _i64, _int, _vp]),
    "ffps_d2h_prefix": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _vp]),
    "ffps_last_launch_count": (_i64, []),
    "ffps_last_error": (ctypes.c_char_p, []),
    "ffps_abi_version": (_int, []),
}


def load():
    """Load (once) and return the ctypes library; raises KernelError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise KernelError(
                    f"CUDA library not built: {LIB_PATH} is missing "
                    "(run __graft_entry__.build() or make -C paper_2604_17720_b200/csrc)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.ffps_abi_version() != 1:
                raise KernelError("ABI version mismatch")
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().ffps_last_error().decode(errors="replace")
        raise KernelError(f"{what} failed ({_STATUS.get(rc, rc)}): {msg}")


def run_kernel(dtype, xyz, batch, cloud_stride, n, iters, seed_pos, index_map, map_stride,
               order, sel_d2, out_stride, stream, algo: str = "auto", stats=None) -> int:
    """``stats``: None or a device pointer to [batch][STATS_WORDS] int64 zeros
    (per-cloud counters of the grid schedule, ffps_run_kernel_stats)."""
    lib = load()
    if stats is None:
        rc = lib.ffps_run_kernel_ex(dtype, xyz, batch, cloud_stride, n, iters, seed_pos,
                                    index_map, map_stride, order, sel_d2, out_stride, stream,
                                    ALGO[algo])
    else:
        rc = lib.ffps_run_kernel_stats(dtype, xyz, batch, cloud_stride, n, iters, seed_pos,
                                       index_map, map_stride, order, sel_d2, out_stride, stream,
                                       ALGO[algo], stats)
    check(rc, "ffps_run_kernel")
    return int(lib.ffps_last_launch_count())


def hierarchical_sample(dtype, xyz, batch, cloud_stride, n, budgets, k, c, fill_mode, pcg_state,
                        cache_enabled, seed_pos, orders, sels, stream) -> int:
    """ffps_hierarchical_sample: ``orders``/``sels`` are per-layer device
    pointers (None where not written); ``pcg_state`` = (state, inc) or None."""
    lib = load()
    L = len(budgets)
    b = (_i64 * L)(*budgets)
    if pcg_state is not None:
        m64 = (1 << 64) - 1
        st, inc = pcg_state
        pcg = (ctypes.c_uint64 * 4)((st >> 64) & m64, st & m64, (inc >> 64) & m64, inc & m64)
    else:
        pcg = None
    o = (_vp * L)(*orders)
    s = (_vp * L)(*sels)
    check(lib.ffps_hierarchical_sample(dtype, xyz, batch, cloud_stride, n, b, L, k, c, fill_mode,
                                       pcg, int(bool(cache_enabled)), seed_pos, o, s, stream),
          "ffps_hierarchical_sample")
    return int(lib.ffps_last_launch_count())


def trim_scratch() -> None:
    """Return the library's cached scratch memory to the driver."""
    check(load().ffps_trim_scratch(), "ffps_trim_scratch")


def fill_slice(dtype, order, sel_d2, batch, out_stride, k, m1, stream) -> int:
    lib = load()
    check(lib.ffps_fill_slice(dtype, order, sel_d2, batch, out_stride, k, m1, stream),
          "ffps_fill_slice")
    return int(lib.ffps_last_launch_count())


def fill_random(dtype, order, sel_d2, batch, out_stride, n, k, m1, pcg_state, stream) -> int:
    """pcg_state = (state, inc) of np.random.PCG64(seed) as Python ints."""
    lib = load()
    st, inc = pcg_state
    m64 = (1 << 64) - 1
    check(lib.ffps_fill_random(dtype, order, sel_d2, batch, out_stride, n, k, m1,
                               (st >> 64) & m64, st & m64, (inc >> 64) & m64, inc & m64, stream),
          "ffps_fill_random")
    return int(lib.ffps_last_launch_count())


def coverage(dtype, xyz, batch, cloud_stride, n, idx, idx_stride, m, out_d2, stream) -> int:
    lib = load()
    check(lib.ffps_coverage(dtype, xyz, batch, cloud_stride, n, idx, idx_stride, m, out_d2,
                            stream), "ffps_coverage")
    return int(lib.ffps_last_launch_count())


def plan(dtype: int, n: int, batch: int) -> dict:
    lib = load()
    out = (ctypes.c_int64 * 7)()
    check(lib.ffps_plan(dtype, n, batch, out), "ffps_plan")
    keys = ("threads", "reg_slots", "smem_slots", "spill_slots", "cluster",
            "ctas_per_sm", "max_clusters")
    return dict(zip(keys, (int(v) for v in out)))


def bucket_plan(dtype: int, n: int) -> dict:
    lib = load()
    out = (ctypes.c_int64 * 4)()
    check(lib.ffps_bucket_plan(dtype, n, out), "ffps_bucket_plan")
    keys = ("threads", "bucket_points", "buckets", "buckets_per_thread")
    return dict(zip(keys, (int(v) for v in out)))


def auto_schedule(n: int, batch: int, dtype: int = F32) -> str:
    """The schedule AUTO picks for a whole batch ("small", "stream", "bucket"
    or "grid@c", c = CTAs per cloud chosen for the whole batch) under the
    arithmetic of ``dtype`` (F32, F64 or F32_F64)."""
    names = {v: k for k, v in ALGO.items()}
    return names[int(load().ffps_auto_schedule_ex(n, batch, dtype))]


def grid_plan(dtype: int, n: int, batch: int, sched: str = "auto") -> dict:
    """K1g configuration for a batch under ``sched`` ("auto" or "grid@c"):
    CTAs per cloud, points per lane (bucket = 32 x ppl points), buckets per
    cloud, dynamic shared memory per CTA."""
    out = (ctypes.c_int64 * 4)()
    check(load().ffps_grid_plan(dtype, n, batch, ALGO[sched], out), "ffps_grid_plan")
    return dict(zip(("cl", "ppl", "buckets", "smem"), (int(v) for v in out)))


def h2d_prefix(dst, src_host, batch, n_prefix, cloud_stride, dtype, stream) -> None:
    check(load().ffps_h2d_prefix(dst, src_host, batch, n_prefix, cloud_stride, dtype, stream),
          "ffps_h2d_prefix")


def d2h_prefix(dst_host, dst_stride, src, src_stride, batch, n_prefix, elem_bytes,
               stream) -> None:
    check(load().ffps_d2h_prefix(dst_host, dst_stride, src, src_stride, batch, n_prefix,
                                 elem_bytes, stream), "ffps_d2h_prefix")
