"""The restatement of the seeded random budget fill (oracle/npchoice.py) is
pinned against NumPy's own Generator.choice and against the reference's
golden prune cases with FillMode.SEEDED_RANDOM (fps_prune.py:101-103)."""

import numpy as np
import pytest

from oracle import npchoice

# (pop, size): both branches (tail shuffle when pop > 10000 and size > pop // 50,
# else Floyd + shuffle), the cut-offs on either side, pop == size
CASES = [(1, 1), (10, 3), (10, 10), (100, 1), (3000, 2999), (10000, 3000), (10001, 200),
         (10001, 201), (10001, 10001), (20000, 400), (20000, 401), (187500, 37500)]


@pytest.mark.parametrize("pop,size", CASES)
def test_restatement_matches_numpy(pop, size):
    for seed in (0, 1, 12345):
        st, inc = npchoice.pcg64_seed_state(seed)
        mine = npchoice.choice_idx(pop, size, st, inc)
        ref = np.random.default_rng(seed).choice(pop, size=size, replace=False)
        assert mine == ref.tolist(), (pop, size, seed)
        pool = np.arange(pop) * 3 + 7  # choice over an array returns pool[idx]
        ref2 = np.random.default_rng(seed).choice(pool, size=size, replace=False)
        assert ref2.tolist() == [3 * v + 7 for v in mine]


@pytest.mark.parametrize("pop,size,seed", [(187500, 37500, 3), (3_000_000, 50_000, 0)])
def test_lemire_rejection_path(pop, size, seed):
    """Cases whose bounded draws hit Lemire's rejection loop (tail and Floyd)."""
    st, inc = npchoice.pcg64_seed_state(seed)
    g = npchoice.PCG64(st, inc)
    mine = npchoice.choice_idx(pop, size, st, inc, g)
    assert g.rejections > 0
    assert mine == np.random.default_rng(seed).choice(pop, size=size, replace=False).tolist()


def test_seeded_fill_matches_reference_goldens(golden):
    cases = [c for c in golden.cases("prune") if c["fill"] == "random"]
    assert cases
    for c in cases:
        k, n = c["fill_boundary"], c["cloud"]["n"]
        want = golden.out(c, "indices")
        got = npchoice.seeded_fill(want[:k], n, c["m1"] - k, c["rng_seed"])
        assert got == want[k:].tolist(), c["id"]
