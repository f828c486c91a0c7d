"""Host-side logic of the round-2 API additions, on CPU (no kernels run):
the arithmetic selector, the divergence report of bench.py, the verify
port's trial generators and the PNN adapter's argument checks."""

import numpy as np
import pytest
import torch

import bench
from paper_2604_17720_b200 import batched, pnn
from paper_2604_17720_b200 import verify as V


def test_precision_selects_the_result_dtype():
    f32 = torch.zeros((1, 4, 3), dtype=torch.float32)
    f64 = f32.double()
    assert batched._out_dtype(f32, None) == torch.float32
    assert batched._out_dtype(f32, "f64") == torch.float64
    assert batched._out_dtype(f32, torch.float64) == torch.float64
    assert batched._out_dtype(f64, None) == torch.float64
    assert batched._out_dtype(f64, "f64") == torch.float64
    with pytest.raises(ValueError):
        batched._out_dtype(f64, "f32")   # would round the cloud
    with pytest.raises(ValueError):
        batched._out_dtype(f32, "f16")


def test_divergence_report():
    a = torch.tensor([[0, 5, 3, 1], [2, 4, 6, 8], [1, 2, 3, 4]])
    b = torch.tensor([[0, 5, 3, 1], [2, 6, 4, 9], [1, 2, 3, 4]])
    d = bench.divergence(a, b, 10)
    assert d["identical_clouds"] == 2 and d["clouds"] == 3 and d["k"] == 4
    assert d["first_divergence"] == [-1, 1, -1]
    assert d["mismatched_positions"] == [0, 3, 0]
    assert d["set_overlap"] == [1.0, 0.75, 1.0]


def test_verify_generators_are_deterministic_and_shaped():
    for kind in ("uniform", "clusters", "sphere"):
        a = V._generate(kind, 257, 11)
        assert a.shape == (257, 3) and a.dtype == np.float64
        assert np.array_equal(a, V._generate(kind, 257, 11))
    s = V._generate("sphere", 1000, 3)
    assert np.allclose(np.sqrt((s * s).sum(1)), 1.0)
    rng = np.random.default_rng(0)
    c = V._trial_cloud("uniform+dups", 100, 5, rng)
    assert c.n == 100 and np.unique(c.points, axis=0).shape[0] <= 50
    r = V.SuiteResult("x", 3, 3)
    assert r.ok and not V.SuiteResult("x", 3, 2).ok


def test_pnn_adapter_rejects_host_and_misshaped_tensors():
    with pytest.raises(TypeError):
        pnn.furthest_point_sample(torch.zeros((1, 10, 3)), 4)
    with pytest.raises(TypeError):
        pnn.flashfps_hierarchy(np.zeros((1, 10, 3)), (4, 2))
