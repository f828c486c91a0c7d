"""Host-side FPS-Cache layer on CPU (no device work): layer budgets, the
footprint model, prefix reuse and the FPSC v1 wire format, mirroring the
reference's tests/test_fps_cache.py host tests, plus byte-for-byte equality
with FPSC blobs written by the unmodified reference (tests/golden)."""

import numpy as np
import pytest

import paper_2604_17720_b200 as ffps
from paper_2604_17720_b200.errors import (BudgetOutOfRange, BudgetsNotMonotone,
                                          PrefixTooLong, UnsupportedFormat)


def _cache_from_golden(golden, c):
    pts = golden.points(c)
    sample = ffps.OrderedSample(golden.out(c, "indices"), golden.out(c, "sel"),
                                fill_boundary=c["fill_boundary"])
    return ffps.CacheRecord.from_sample(ffps.PointCloud(pts), sample), sample


def test_layer_budgets_validation():  # reference test_fps_cache.py:26-34
    assert ffps.LayerBudgets((8, 4, 2)).budgets == (8, 4, 2)
    assert len(ffps.LayerBudgets((3,))) == 1
    with pytest.raises(BudgetsNotMonotone):
        ffps.LayerBudgets((4, 8))
    with pytest.raises(BudgetsNotMonotone):
        ffps.LayerBudgets(())
    with pytest.raises(BudgetOutOfRange):
        ffps.LayerBudgets((4, 0))


def test_footprint_model():  # reference test_fps_cache.py:131-140
    assert ffps.BYTES_PER_ENTRY == 36
    assert ffps.cache_footprint(1) == 36
    for m in (1, 2, 17, 1000, 72_250):
        assert ffps.cache_footprint(2 * m) == 2 * ffps.cache_footprint(m)
    assert ffps.cache_footprint(72_250) == 2_601_000
    with pytest.raises(BudgetOutOfRange):
        ffps.cache_footprint(0)


def test_fpsc_bytes_match_reference(golden):
    cases = golden.cases("fpsc")
    assert len(cases) >= 3
    for c in cases:
        cache, sample = _cache_from_golden(golden, c)
        blob = cache.to_bytes()
        want = golden.out(c, "blob").tobytes()
        assert blob == want, c["id"]
        assert len(blob) - 16 == cache.footprint_bytes == c["footprint"]
        back = ffps.CacheRecord.from_bytes(want)
        assert np.array_equal(back.layer1.indices, sample.indices)
        assert np.array_equal(back.layer1.selection_dist2, sample.selection_dist2)
        assert back.layer1.fill_boundary == c["back_fill_boundary"]
        assert np.array_equal(back.points, cache.points)


def test_prefix_reuse_and_files(golden, tmp_path):  # reference :84-95, :151-180
    c = golden.cases("fpsc")[0]
    cache, sample = _cache_from_golden(golden, c)
    for m in (1, 7, len(sample)):
        pre = ffps.prefix_reuse(cache, m)
        assert np.array_equal(pre.indices, sample.indices[:m])
        assert pre.fill_boundary == min(sample.fill_boundary, m)
    with pytest.raises(PrefixTooLong):
        ffps.prefix_reuse(cache, len(sample) + 1)
    with pytest.raises(PrefixTooLong):
        ffps.prefix_reuse(cache, 0)
    ffps.write_cache(cache, tmp_path / "l1.cache")
    back = ffps.read_cache(tmp_path / "l1.cache")
    assert np.array_equal(back.layer1.indices, sample.indices)
    ffps.write_cache_text(cache, tmp_path / "l1.txt")
    lines = (tmp_path / "l1.txt").read_text().splitlines()
    assert f"count={len(sample)}" in lines[0] and f"fill_boundary={sample.fill_boundary}" in lines[0]
    for i, line in enumerate(lines[1:]):
        idx, x, y, z, d2 = line.split()
        assert int(idx) == sample.indices[i] and float(d2) == sample.selection_dist2[i]
        assert (float(x), float(y), float(z)) == tuple(cache.points[i])


def test_corrupt_blobs_rejected(golden):  # reference :182-191
    c = golden.cases("fpsc")[0]
    blob = golden.out(c, "blob").tobytes()
    with pytest.raises(UnsupportedFormat):
        ffps.CacheRecord.from_bytes(b"JUNK" + blob[4:])
    with pytest.raises(UnsupportedFormat):
        ffps.CacheRecord.from_bytes(blob[:-5])
    with pytest.raises(UnsupportedFormat):
        ffps.CacheRecord.from_bytes(b"FP")
