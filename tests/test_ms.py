"""MS — bottom-up merge sort (no reference code):
ir/merge_step.ir run to a fixpoint per pass by the reference interpreter pins
the oracle restatement (golden fixtures, oracle/gen_golden.py), and — on the
GPU — both forms of csrc/merge_sort.cu against it."""
import numpy as np
import pytest

from conftest import load_golden

import paper_2107_05681_b200 as darm


def test_merge_restatement_matches_reference_golden(restatement):
    gold = load_golden("merge_sort.json")
    for case in gold["cases"]:
        keys = np.array(case["keys"], dtype=np.int32)
        restatement.merge_sort(keys)
        assert keys.tolist() == case["sorted"], case["n"]


def test_merge_melded_spec_is_the_reference_pass_output():
    """runDarm melds the take-left / take-right arms block-block (one select of
    the run index); at full warps the reference simulator sees fewer
    serialized cycles after it."""
    gold = load_golden("merge_sort.json")
    assert [(m["kind"], m["selectsInserted"]) for m in gold["melds"]] == [("block-block", 1)]
    big = [c for c in gold["cases"] if c["n"] >= 256]
    for case in big:
        u, m = case["stats_unit_latency"]["unmelded"], case["stats_unit_latency"]["melded"]
        assert m[3] < u[3]


@pytest.mark.parametrize("n", [0, 1, 2, 5, 2047, 2048, 2049, 10000, 1 << 16])
def test_merge_restatement_sorts(restatement, n):
    rng = np.random.default_rng(n)
    keys = rng.integers(-(2 ** 31), 2 ** 31, size=n, dtype=np.int64).astype(np.int32)
    want = np.sort(keys)
    restatement.merge_sort(keys)
    assert (keys == want).all()


@pytest.mark.gpu
def test_merge_gpu_golden():
    gold = load_golden("merge_sort.json")
    for case in gold["cases"]:
        for variant in (0, 1):
            keys = np.array(case["keys"], dtype=np.int32)
            darm.merge_sort(keys, variant)
            assert keys.tolist() == case["sorted"], (case["n"], variant)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 2, 7, 2047, 2048, 2049, 4095, 4096, 4097, 6145, 8193, 100003, 1 << 20, (1 << 22) + 37])
def test_merge_gpu_vs_restatement(restatement, n):
    import torch

    rng = np.random.default_rng(n + 5)
    for dup in (False, True):
        lo, hi = (-16, 17) if dup else (-(2 ** 31), 2 ** 31)
        keys = rng.integers(lo, hi, size=n, dtype=np.int64).astype(np.int32)
        want = keys.copy()
        restatement.merge_sort(want)
        for variant in (0, 1):
            k = torch.from_numpy(keys.copy()).cuda()
            darm.merge_sort(k, variant)
            assert (k.cpu().numpy() == want).all(), (n, dup, variant)


@pytest.mark.gpu
def test_merge_gpu_extremes_and_host_mode():
    keys = np.array([2 ** 31 - 1, -(2 ** 31), 0, -1, 1, 2 ** 31 - 1, -(2 ** 31)] * 1000, dtype=np.int32)
    want = np.sort(keys)
    for variant in (0, 1):
        k = keys.copy()
        st = darm.merge_sort(k, variant)
        assert (k == want).all()
        assert st["launches"] == 1 + 1          # tile pass (widths < 4096) + width 4096
