"""Device plumbing between torch tensors and the C ABI.

torch provides device memory, pinned host memory and streams; every FLOP of
the hot path runs in the library's own kernels (K1 greedy, K2 fill).  The
launch counter lets benches report how many of those kernels ran.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .errors import KernelError

_DTYPE_CODE = {torch.float32: _native.F32, torch.float64: _native.F64}
_launches = 0
_timers: list | None = None
_stats: list | None = None
_algo = "auto"


def current_schedule() -> str:
    return _algo


def set_schedule(name: str) -> str:
    """Select the greedy schedule for subsequent calls: "auto" (default),
    "bucket" (K0+K1b, bounded re-evaluation) or "stream" (K1, every point every
    iteration).  Results are identical; returns the previous setting."""
    global _algo
    if name not in _native.ALGO:
        raise ValueError(f"unknown schedule {name!r}; expected one of {sorted(_native.ALGO)}")
    prev, _algo = _algo, name
    return prev


class kernel_timer:
    """Context manager that brackets every K1 (greedy) launch issued inside it
    with CUDA events on the launching stream; ``records`` holds
    (batch, n, iters, start, end) tuples.  Used by bench.py to time the
    dominant kernel live, inside the timed region."""

    def __enter__(self):
        global _timers
        self.records = []
        _timers = self.records
        return self

    def __exit__(self, *exc):
        global _timers
        _timers = None
        return False

    def kernel_ms(self):
        return [(b, n, it, s.elapsed_time(e)) for b, n, it, s, e in self.records]


class grid_stats:
    """Context manager that attaches a per-cloud counter block to every greedy
    launch issued inside it (ffps_run_kernel_stats); ``records`` holds
    (batch, n, iters, stats) with stats a (batch, 4) int64 device tensor:
    rounds, loop cycles on cluster rank 0, re-evaluated buckets, rounds
    ranked through the general path, summed over the cluster's CTAs (grid
    schedule only; zeros otherwise)."""

    def __enter__(self):
        global _stats
        self.records = []
        _stats = self.records
        return self

    def __exit__(self, *exc):
        global _stats
        _stats = None
        return False


def launches() -> int:
    """Kernel launches issued by this process so far (K1 + K2)."""
    return _launches


def _count(n: int) -> None:
    global _launches
    _launches += n


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise KernelError("no CUDA device is available; the FlashFPS path has no CPU fallback")
    _native.load()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
        else torch.device(device)
    if dev.type != "cuda":
        raise KernelError(f"device {dev} is not a CUDA device")
    return dev


def dtype_code(t: torch.Tensor, out: torch.Tensor | None = None) -> int:
    """ABI dtype of coordinates ``t`` with results ``out`` (default: same
    dtype): float32 coordinates with float64 results select FFPS_F32_F64,
    binary64 arithmetic on float coordinates."""
    try:
        code = _DTYPE_CODE[t.dtype]
    except KeyError:
        raise TypeError(f"coordinates must be float32 or float64, got {t.dtype}") from None
    if out is not None and out.dtype != t.dtype:
        if t.dtype == torch.float32 and out.dtype == torch.float64:
            return _native.F32_F64
        raise TypeError(f"{t.dtype} coordinates cannot produce {out.dtype} distances")
    return code


def _stream_handle(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def greedy(xyz: torch.Tensor, n: int, iters: int, seeds: torch.Tensor,
           order: torch.Tensor, sel: torch.Tensor, index_map: torch.Tensor | None = None,
           stream=None) -> None:
    """K1 over a batch: xyz (B, N, 3) CUDA, contiguous; writes order[:, :iters]
    and sel[:, :iters] (row stride = order.stride(0))."""
    B = xyz.shape[0]
    if B == 0:
        return
    assert xyz.is_cuda and xyz.is_contiguous() and xyz.dim() == 3 and xyz.shape[2] == 3
    assert order.dtype == torch.int64 and order.stride(1) == 1 and sel.stride(1) == 1
    assert sel.stride(0) == order.stride(0)
    code = dtype_code(xyz, sel)
    assert seeds.dtype == torch.int64 and seeds.is_cuda and seeds.numel() == B
    map_ptr, map_stride = None, 0
    if index_map is not None:
        assert index_map.dtype == torch.int64 and index_map.stride(1) == 1
        map_ptr, map_stride = index_map.data_ptr(), index_map.stride(0)
    with torch.cuda.device(xyz.device):
        if _timers is not None:
            strm = torch.cuda.current_stream() if stream is None else stream
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(strm)
        st_ptr = None
        if _stats is not None:
            st_t = torch.zeros((B, _native.STATS_WORDS), dtype=torch.int64, device=xyz.device)
            _stats.append((B, n, iters, st_t))
            st_ptr = st_t.data_ptr()
        _count(_native.run_kernel(code, xyz.data_ptr(), B, xyz.shape[1], n, iters,
                                  seeds.data_ptr(), map_ptr, map_stride, order.data_ptr(),
                                  sel.data_ptr(), order.stride(0), _stream_handle(stream),
                                  _algo, st_ptr))
        if _timers is not None:
            ev1.record(strm)
            _timers.append((B, n, iters, ev0, ev1))


def fill_slice(order: torch.Tensor, sel: torch.Tensor, k: int, m1: int, stream=None) -> None:
    """K2: order[:, k:m1] <- first ascending unselected indices, sel[:, k:m1] <- 0."""
    B = order.shape[0]
    if B == 0 or m1 <= k:
        return
    with torch.cuda.device(order.device):
        _count(_native.fill_slice(dtype_code(sel), order.data_ptr(), sel.data_ptr(), B,
                                  order.stride(0), k, m1, _stream_handle(stream)))


def fill_random(order: torch.Tensor, sel: torch.Tensor, n: int, k: int, m1: int, rng_seed: int,
                stream=None) -> None:
    """K2r: order[:, k:m1] <- np.random.default_rng(rng_seed).choice(pool, m1 - k,
    replace=False) of each cloud's unselected indices, sel[:, k:m1] <- 0.  Only
    the generator's seeding (SeedSequence -> PCG64 state) runs on the host."""
    B = order.shape[0]
    if B == 0 or m1 <= k:
        return
    st = np.random.PCG64(rng_seed).state["state"]
    with torch.cuda.device(order.device):
        _count(_native.fill_random(dtype_code(sel), order.data_ptr(), sel.data_ptr(), B,
                                   order.stride(0), n, k, m1,
                                   (int(st["state"]), int(st["inc"])), _stream_handle(stream)))


def seeds_tensor(seed_index, B: int, device) -> torch.Tensor:
    """(B,) int64 seed positions on ``device``, stream-ordered (no host sync
    when every cloud starts from the same position)."""
    arr = np.broadcast_to(np.asarray(seed_index, dtype=np.int64), (B,))
    if B > 0 and (arr == arr[0]).all():
        return torch.full((B,), int(arr[0]), dtype=torch.int64, device=device)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device, non_blocking=False)


def coverage(xyz: torch.Tensor, idx: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    """K0 x2 + K5: out[b] = max_p min_s d2(p, s) over xyz[b] and xyz[b][idx[b]]."""
    B = xyz.shape[0]
    if B == 0:
        return
    assert xyz.is_cuda and xyz.is_contiguous() and idx.dtype == torch.int64
    assert idx.stride(1) == 1 and out.is_contiguous()
    code = dtype_code(xyz, out)
    with torch.cuda.device(xyz.device):
        _count(_native.coverage(code, xyz.data_ptr(), B, xyz.shape[1], xyz.shape[1],
                                idx.data_ptr(), idx.stride(0), idx.shape[1], out.data_ptr(),
                                _stream_handle(stream)))
