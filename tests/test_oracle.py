"""The CPU oracle (test infrastructure) pinned against the reference's own
golden vectors (tests/golden, produced by the unmodified reference)."""

import numpy as np
import pytest

from oracle import oracle


def _ids(cases):
    return [c["id"] for c in cases]


def test_golden_manifest_is_complete(golden):
    ops = {c["op"] for c in golden.cases()}
    assert {"fps", "prune", "hier", "prefix", "fps32"} <= ops
    assert len(golden.cases()) >= 80


def test_oracle_fps_matches_reference(golden):
    for c in golden.cases("fps"):
        pts = golden.points(c)
        idx, sel, evals = oracle.run_kernel(pts, c["m"], c["seed"])
        assert np.array_equal(idx, golden.out(c, "indices")), c["id"]
        assert np.array_equal(sel, golden.out(c, "sel")), c["id"]
        assert evals == c["stats"][0]


def test_oracle_fp32_matches_numpy_f32_restatement(golden):
    for c in golden.cases("fps32"):
        pts = golden.points(c).astype(np.float32)
        idx, sel, _ = oracle.run_kernel(pts, c["m"], c["seed"])
        assert sel.dtype == np.float32
        assert np.array_equal(idx, golden.out(c, "indices")), c["id"]
        assert np.array_equal(sel, golden.out(c, "sel")), c["id"]


def test_oracle_prune_slice_matches_reference(golden):
    n_checked = 0
    for c in golden.cases("prune"):
        if c["fill"] != "slice":
            continue
        idx, sel, k, cc = oracle.fps_prune(golden.points(c), c["m1"], c["p"], c["seed"])
        assert k == c["fill_boundary"] == c["stats"][1], c["id"]
        assert cc == c["stats"][2]
        assert np.array_equal(idx, golden.out(c, "indices")), c["id"]
        assert np.array_equal(sel, golden.out(c, "sel")), c["id"]
        n_checked += 1
    assert n_checked >= 10


def test_oracle_hierarchy_matches_reference(golden):
    for c in golden.cases("hier"):
        layers = oracle.hierarchical(golden.points(c), c["budgets"], c["p"], c["seed"],
                                     c["cache"])
        for li, (idx, sel) in enumerate(layers):
            assert np.array_equal(idx, golden.out(c, f"L{li}_indices")), (c["id"], li)
            assert np.array_equal(sel, golden.out(c, f"L{li}_sel")), (c["id"], li)


def test_collinear_worked_example():
    # test_fps_core.py:34-41 / fps_prune.py trace test_fps_prune.py:55-63
    pts = np.array([(0, 0, 0), (1, 0, 0), (2, 0, 0), (3, 0, 0), (10, 0, 0)], float)
    idx, sel, ev = oracle.run_kernel(pts, 5, 0)
    assert idx.tolist() == [0, 4, 3, 1, 2]
    assert sel[1:].tolist() == [100.0, 9.0, 1.0, 1.0] and np.isinf(sel[0])
    assert ev == 20
    idx, sel, k, c = oracle.fps_prune(pts, 4, 0.5)
    assert idx.tolist() == [0, 1, 2, 3] and k == 2 and c == 2
    assert sel.tolist()[1:] == [1.0, 0.0, 0.0]


@pytest.mark.parametrize("p,m1,want", [(0.3, 90, 62), (0.8, 5, 1), (0.9, 6000, 599),
                                       (0.75, 50000, 12500), (0.75, 75000, 18750),
                                       (0.75, 1, 1), (0.75, 50, 12)])
def test_kernel_budget_ieee_floor(p, m1, want):
    # fps_prune.py:45-47 computes floor((1.0 - p) * m1) in binary64
    assert oracle.kernel_budget(p, m1) == want


def test_oracle_batch_threads_identical():
    rng = np.random.default_rng(3)
    xyz = rng.random((6, 2000, 3)).astype(np.float32)
    o1, s1 = oracle.run_kernel_batch(xyz, 300, 0, threads=1)
    o4, s4 = oracle.run_kernel_batch(xyz, 300, 0, threads=4)
    assert np.array_equal(o1, o4) and np.array_equal(s1, s4)
    for b in range(6):
        idx, sel, _ = oracle.run_kernel(xyz[b], 300, 0)
        assert np.array_equal(o1[b], idx) and np.array_equal(s1[b], sel)
