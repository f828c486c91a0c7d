"""Adversarial point distributions for the exact-skip arguments.

The multi-winner and bucketed schedules (K1g, K1b) skip buckets through
rounded lower bounds (RN monotonicity, DESIGN §3 K1b / K1g) and, under
binary64 on float coordinates, through binary32 bounds rounded down against
keys rounded up.  Spatial indexing is outside the reference's own scope
(SPEC.md:130), so these tests aim at the places such bounds break: extreme
density contrast, degenerate (flat) bucket boxes, large offsets that make
coordinate differences round, near-duplicates one ulp apart, wide dynamic
ranges, and squares that overflow binary32.  Bar: indices and selection
distances bit-identical to the CPU oracle (pinned to the reference) under
every schedule and arithmetic."""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2604_17720_b200 import _device
from test_gpu_parity import _Sched

pytestmark = pytest.mark.gpu


def _adversarial(kind: str, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "core_shell":        # 90% in a 1e-4 ball, 10% on a radius-1e3 sphere
        core = rng.normal(size=(n - n // 10, 3)) * 1e-4
        v = rng.normal(size=(n // 10, 3))
        shell = v / np.linalg.norm(v, axis=1, keepdims=True) * 1e3
        pts = np.vstack([core, shell])[rng.permutation(n)]
    elif kind == "line":            # zero extent in two axes
        pts = np.zeros((n, 3))
        pts[:, 0] = np.cumsum(rng.exponential(size=n))
        pts = pts[rng.permutation(n)]
    elif kind == "plane_grid":      # a flat integer lattice: massive exact ties
        side = int(np.ceil(np.sqrt(n)))
        g = np.stack(np.meshgrid(np.arange(side), np.arange(side), indexing="ij"), -1)
        g = g.reshape(-1, 2)[rng.permutation(side * side)[:n]]
        pts = np.column_stack([g, np.full(n, 7.0)])
    elif kind == "big_offset":      # 1e-3 cube at 1e5: differences round in binary32
        pts = 1e5 + rng.random((n, 3)) * 1e-3
    elif kind == "log_radii":       # radii log-uniform over 1e-6 .. 1e3
        v = rng.normal(size=(n, 3))
        r = 10.0 ** rng.uniform(-6, 3, size=n)
        pts = v / np.linalg.norm(v, axis=1, keepdims=True) * r[:, None]
    elif kind == "ulp_pairs":       # pairs one float32 ulp apart
        base = rng.random((n // 2, 3)).astype(np.float32)
        twin = np.nextafter(base, np.float32(2.0))
        pts = np.vstack([base, twin])[rng.permutation(2 * (n // 2))]
        if pts.shape[0] < n:
            pts = np.vstack([pts, pts[:1]])
    elif kind == "overflow":        # |x| ~ 1e20: squares overflow binary32 to +inf
        pts = rng.uniform(-1e20, 1e20, size=(n, 3))
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(pts, dtype=np.float64)


KINDS = ["core_shell", "line", "plane_grid", "big_offset", "log_radii", "ulp_pairs", "overflow"]
SCHEDS = ["grid@1", "grid@2", "grid@4", "bucket", "stream", "small"]


def _run(x, m, precision):
    B = x.shape[0]
    xd = torch.from_numpy(x).cuda()
    order = torch.empty((B, m), dtype=torch.int64, device="cuda")
    sel = torch.empty((B, m), dtype=torch.float64 if precision == "f64" else xd.dtype,
                      device="cuda")
    _device.greedy(xd, x.shape[1], m, _device.seeds_tensor(np.zeros(B, np.int64), B, "cuda"),
                   order, sel)
    return order.cpu().numpy(), sel.cpu().numpy()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("arith", ["f32", "f32_f64", "f64"])
def test_adversarial_clouds_bit_exact(cuda, kind, sched, arith):
    for n, m in [(3000, 900), (24000, 1500), (60000, 3000)]:
        if sched == "small" and n > 8192:
            continue
        pts = np.stack([_adversarial(kind, n, s) for s in (1, 2)])
        if arith == "f64":
            x, want_x, prec = pts, pts, None
        else:
            x = pts.astype(np.float32)
            want_x = x.astype(np.float64) if arith == "f32_f64" else x
            prec = "f64" if arith == "f32_f64" else None
        with _Sched(sched):
            go, gs = _run(x, m, prec)
        wo, ws = oracle.run_kernel_batch(want_x, m, np.zeros(2, np.int64))
        for b in range(2):
            bad = np.flatnonzero(go[b] != wo[b])
            assert bad.size == 0, f"{kind} n={n} cloud {b}: first divergence at {bad[0]}"
            assert np.array_equal(gs[b], ws[b]), f"{kind} n={n} cloud {b}: distances differ"
