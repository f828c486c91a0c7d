import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


class Golden:
    """Golden vectors produced by the unmodified reference (make_golden.py)."""

    def __init__(self):
        with open(os.path.join(GOLDEN, "manifest.json")) as fh:
            self.meta = json.load(fh)
        self.arrays = np.load(os.path.join(GOLDEN, "golden.npz"))

    def cases(self, op=None):
        return [c for c in self.meta["cases"] if op is None or c["op"] == op]

    def points(self, case):
        from clouds import digest, make_cloud
        if "literal" in case:
            return self.arrays[case["literal"]]
        cl = case["cloud"]
        pts = make_cloud(cl["kind"], cl["n"], cl["seed"])
        assert digest(pts) == cl["sha"], "cloud generator drifted; regenerate goldens"
        return pts

    def out(self, case, key):
        return self.arrays[case["outputs"][key]]


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is available")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)
