"""GPU parity for N-Queens (NQU): per-prefix solution counts bit-exact against the
reference-interpreted IR chain (small n) and the C restatement, and the
published totals (OEIS A000170) at the BASELINE size n = 16."""
import numpy as np
import pytest

from conftest import load_golden
from test_oracle import NQUEENS

import paper_2107_05681_b200 as darm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch

    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    darm.init()


@pytest.mark.parametrize("variant", [0, 1])
def test_nqueens_reference_chain_golden(variant):
    gold = load_golden("nqueens_chain.json")
    for case in gold["cases"]:
        sols, per, _ = darm.nqueens(case["n"], case["base"], variant, per_prefix=True)
        assert per.tolist() == case["per_prefix"], (case["n"], variant)
        assert sols == case["solutions"]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("n,base", [(10, 3), (12, 4), (13, 5), (14, 4)])
def test_nqueens_per_prefix_vs_restatement(restatement, variant, n, base):
    states = restatement.nqueens_prefixes(n, base)
    tot, want, _ = restatement.nqueens_count(n, base, states)
    sols, per, _ = darm.nqueens(n, base, variant, per_prefix=True)
    assert (per == want).all()
    assert sols == tot == NQUEENS[n]


@pytest.mark.parametrize("variant", [0, 1])
def test_nqueens_config3_n16(variant):
    """BASELINE config 3: N=16, prefix search space (6-row prefixes)."""
    sols, _, st = darm.nqueens(16, 6, variant)
    assert sols == 14772512


def test_nqueens_rank_partition():
    """Prefixes dealt round-robin over 3 'ranks' sum to the total (the
    multi-GPU decomposition, one call per rank)."""
    parts = [darm.nqueens(13, 4, 1, rank=r, world=3)[0] for r in range(3)]
    assert sum(parts) == NQUEENS[13]


def test_nqueens_small_and_edge():
    for n in range(2, 10):
        for base in range(1, n):
            assert darm.nqueens(n, base, 1)[0] == NQUEENS[n], (n, base)
    with pytest.raises(darm.DarmUserError):
        darm.nqueens(8, 8)
    with pytest.raises(darm.DarmUserError):
        darm.nqueens(1, 1)


@pytest.mark.parametrize("variant", [0, 1])
def test_nqueens_mirror_symmetry(variant):
    """DARM_NQ_MIRROR: row-0 queen in the left half (x2) and the middle column of
    an odd board (x1) — the same totals with half the search."""
    for n in range(4, 15):
        for base in (1, 2, min(4, n - 1)):
            assert darm.nqueens(n, base, variant, mirror=True)[0] == NQUEENS[n], (n, base)
    parts = [darm.nqueens(13, 4, variant, rank=r, world=3, mirror=True)[0] for r in range(3)]
    assert sum(parts) == NQUEENS[13]
    assert darm.nqueens(16, 7, variant, mirror=True)[0] == 14772512
    _, per, _ = darm.nqueens(9, 3, variant, per_prefix=True, mirror=True)
    _, per_full, _ = darm.nqueens(9, 3, variant, per_prefix=True)
    assert len(per) < len(per_full)


# ---- the paper's shape: ir/nqueens_step.ir (DARM_NQ_PAPER_SHAPE)
@pytest.mark.parametrize("variant", [0, 1])
def test_nqueens_paper_shape_reference_chain_golden(variant):
    """Both forms of the paper-shaped encoding against the reference
    interpreter running ir/nqueens_step.ir to a fixpoint."""
    gold = load_golden("nqueens_step_chain.json")
    for case in gold["cases"]:
        sols, per, _ = darm.nqueens(case["n"], case["base"], variant, per_prefix=True, paper_shape=True)
        assert per.tolist() == case["per_prefix"], (case["n"], variant)
        assert sols == case["solutions"]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("n,base,mirror", [(10, 3, False), (12, 4, True), (14, 4, False), (14, 5, True)])
def test_nqueens_paper_shape_equals_symmetric(variant, n, base, mirror):
    """Same search, two encodings: per-prefix counts equal, totals = OEIS."""
    a = darm.nqueens(n, base, variant, per_prefix=True, mirror=mirror, paper_shape=True)
    b = darm.nqueens(n, base, variant, per_prefix=True, mirror=mirror)
    assert (a[1] == b[1]).all()
    assert a[0] == b[0] == NQUEENS[n]


@pytest.mark.parametrize("variant", [0, 1])
def test_nqueens_paper_shape_n16(variant):
    assert darm.nqueens(16, 7, variant, mirror=True, paper_shape=True, want_stats=False)[0] == 14772512


def test_nqueens_paper_shape_limits():
    with pytest.raises(darm.DarmUserError):
        darm.nqueens(17, 5, 1, paper_shape=True)
