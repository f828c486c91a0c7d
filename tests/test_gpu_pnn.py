"""The point-network call-site adapter (paper_2604_17720_b200/pnn.py): the
OpenPoints-shaped ``furthest_point_sample`` and the per-stage FlashFPS
hierarchy stay on the device and equal the batched API, the CPU oracle and
the reference's goldens."""

import numpy as np
import pytest
import torch

import paper_2604_17720_b200 as ffps
from oracle import oracle

pytestmark = pytest.mark.gpu


def test_furthest_point_sample_matches_fps_batch_and_oracle(cuda):
    rng = np.random.default_rng(8)
    xyz = torch.from_numpy(rng.random((4, 24000, 3)).astype(np.float32)).cuda()
    idx = ffps.furthest_point_sample(xyz, 6000)
    assert idx.dtype == torch.int32 and idx.is_cuda and idx.shape == (4, 6000)
    ref, _ = ffps.fps_batch(xyz, 6000)
    assert torch.equal(idx.long(), ref.indices)
    wo, _ = oracle.run_kernel_batch(xyz.cpu().numpy(), 6000, np.zeros(4, np.int64))
    assert np.array_equal(idx.cpu().numpy(), wo)
    # binary64 on float coordinates == the binary64 oracle on the upcast cloud
    i64 = ffps.furthest_point_sample(xyz[:, :5000], 1000, precision="f64")
    wo64, _ = oracle.run_kernel_batch(xyz[:, :5000].cpu().numpy().astype(np.float64), 1000,
                                      np.zeros(4, np.int64))
    assert np.array_equal(i64.cpu().numpy(), wo64)
    # a strided (non-contiguous) view is accepted
    big = torch.from_numpy(rng.random((2, 3000, 4)).astype(np.float32)).cuda()
    a = ffps.furthest_point_sample(big[..., :3], 500)
    b = ffps.furthest_point_sample(big[..., :3].contiguous(), 500)
    assert torch.equal(a, b)


def test_furthest_point_sample_reference_goldens(golden, cuda):
    """Seed-0 fps goldens of the unmodified reference, through the adapter
    in the reference's binary64 arithmetic (float64 coordinates)."""
    n = 0
    for c in golden.cases("fps"):
        if c["seed"] != 0:
            continue
        pts = torch.from_numpy(golden.points(c)).cuda().unsqueeze(0)
        idx = ffps.furthest_point_sample(pts, c["m"])
        assert np.array_equal(idx[0].cpu().numpy(), golden.out(c, "indices")), c["id"]
        n += 1
    assert n >= 5


@pytest.mark.parametrize("cache", [True, False])
def test_flashfps_hierarchy_stages(cuda, cache):
    rng = np.random.default_rng(9)
    budgets = (6000, 1500, 375, 93)
    xyz = torch.from_numpy(rng.random((3, 24000, 3)).astype(np.float32)).cuda()
    stages = ffps.flashfps_hierarchy(xyz, budgets, 0.75, cache=cache)
    assert [tuple(s.shape) for s in stages] == [(3, m) for m in budgets]
    layers, _, _ = ffps.hierarchical_sample_batch(xyz, budgets, ffps.PruneConfig(p=0.75), 0,
                                                  cache)
    for s, l in zip(stages, layers):
        assert s.is_cuda and torch.equal(s, l.indices)
    for b in range(3):
        want = oracle.hierarchical(xyz[b].cpu().numpy(), budgets, 0.75, 0, cache)
        for s, (wi, _) in zip(stages, want):
            assert np.array_equal(s[b].cpu().numpy(), wi)
    if cache:  # deeper stages are views of stage 1
        assert stages[1].data_ptr() == stages[0].data_ptr()


def test_adapter_argument_errors(cuda):
    with pytest.raises(TypeError):
        ffps.furthest_point_sample(torch.zeros((1, 10, 3)), 4)   # host tensor
    with pytest.raises(ValueError):
        ffps.furthest_point_sample(torch.zeros((10, 3), device="cuda"), 4)
    with pytest.raises(ffps.errors.BudgetOutOfRange):
        ffps.furthest_point_sample(torch.zeros((1, 10, 3), device="cuda"), 11)
