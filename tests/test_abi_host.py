"""CPU-only checks of the boundary and the host layer (no compute calls):
the C-ABI library loads and exports every symbol include/*.h declares, the
ctypes signatures match the header, the reference's exceptions are raised
before any device requirement, and the product path fails loudly (no CPU
fallback) when no CUDA device is present."""

import ctypes
import glob
import os
import re

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from paper_2604_17720_b200 import _native
from paper_2604_17720_b200.errors import KernelError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ffps_[a-z_0-9]+)\s*\(",
                            src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    declared = _declared()
    assert "ffps_run_kernel" in declared and "ffps_fill_slice" in declared
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/ but not exported"
    assert set(declared) == set(_native.SIGNATURES), "ctypes table out of sync with header"


def test_abi_version_and_argument_errors_without_gpu():
    lib = _native.load()
    assert lib.ffps_abi_version() == 1
    # argument validation happens before any CUDA call
    assert lib.ffps_run_kernel(9, None, 1, 10, 10, 5, None, None, 0, None, None, 5, None) == -1
    assert b"dtype" in lib.ffps_last_error()
    assert lib.ffps_run_kernel(0, 1, 1, 10, 10, 11, 1, None, 0, 1, 1, 11, None) == -1
    assert lib.ffps_fill_slice(0, 1, 1, 1, 10, 5, 4, None) == -1
    assert lib.ffps_run_kernel(0, None, 0, 10, 10, 5, None, None, 0, None, None, 5, None) == 0
    out = (ctypes.c_int64 * 7)()
    assert lib.ffps_plan(0, 0, 1, out) == -1
    assert lib.ffps_grid_plan(7, 1000, 1, 0, out) == -1    # bad dtype, before any CUDA call
    assert lib.ffps_grid_plan(0, 0, 1, 0, out) == -1


def test_reference_errors_precede_device_requirement():
    pts = np.random.default_rng(0).random((2, 100, 3)).astype(np.float32)
    with pytest.raises(ffps.errors.BudgetOutOfRange):
        ffps.fps_batch(pts, 0)
    with pytest.raises(ffps.errors.BudgetOutOfRange):
        ffps.fps_batch(pts, 101)
    with pytest.raises(ffps.errors.SeedOutOfRange):
        ffps.fps_batch(pts, 10, seed_index=100)
    with pytest.raises(ffps.errors.SeedNotInCandidates):
        ffps.fps_prune_batch(pts, 40, ffps.PruneConfig(p=0.5), seed_index=60)
    with pytest.raises(ffps.errors.BudgetExceedsCloud):
        ffps.hierarchical_sample_batch(pts, (200, 50), ffps.PruneConfig())
    with pytest.raises(ffps.errors.BudgetsNotMonotone):
        ffps.hierarchical_sample_batch(pts, (20, 50), ffps.PruneConfig())
    with pytest.raises(ffps.errors.EmptyCloud):
        ffps.validate_cloud(np.zeros((0, 3)))
    with pytest.raises(ffps.errors.NonFiniteCoordinate) as ei:
        ffps.validate_cloud([(0, 0, 0), (1, np.nan, 0)])
    assert ei.value.index == 1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    pts = np.random.default_rng(0).random((50, 3))
    with pytest.raises(KernelError):
        ffps.fps(ffps.PointCloud(pts), 5)
    with pytest.raises(KernelError):
        ffps.hierarchical_sample_batch(pts.astype(np.float32)[None], (8, 4),
                                       ffps.PruneConfig(p=0.5))


@pytest.mark.parametrize("p,m1,k", [(0.3, 90, 62), (0.8, 5, 1), (0.9, 6000, 599),
                                    (0.75, 50000, 12500), (0.0, 7, 7)])
def test_kernel_budget_is_ieee_double(p, m1, k):
    assert ffps.PruneConfig(p=p).kernel_budget(m1) == k


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2604_17720_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True):
        src = open(path).read()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), path
