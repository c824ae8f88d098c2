"""PCM — Batcher odd-even merge sort of buckets (no reference
code): ir/oddeven_step.ir run by the reference interpreter pins the oracle
restatement (golden fixtures, oracle/gen_golden.py), and — on the GPU — both
forms and every keys-per-thread shape of csrc/oddeven_sort.cu against it."""
import numpy as np
import pytest

from conftest import load_golden

import paper_2107_05681_b200 as darm


def test_oddeven_restatement_matches_reference_golden(restatement):
    gold = load_golden("oddeven_sort.json")
    for case in gold["cases"]:
        keys = np.array(case["keys"], dtype=np.int32)
        restatement.oddeven_sort(keys, case["bucket"])
        assert keys.tolist() == case["sorted"], case["bucket"]


def test_oddeven_melded_spec_is_the_reference_pass_output():
    """The melded forms mirror runDarm's output for ir/oddeven_step.ir: a
    block-region meld (the upper region with the idle block, by region
    replication) and a region-region meld (the lower region with the result),
    PAPER.md:947-948.  The reference simulator sees higher lane utilisation
    after it and, with its default latencies (where the melded shared / global
    memory instructions count), fewer serialized cycles from 4-key buckets up."""
    gold = load_golden("oddeven_sort.json")
    assert [m["kind"] for m in gold["melds"]] == ["block-region", "region-region"]
    for case in gold["cases"]:
        u, m = case["stats_unit_latency"]["unmelded"], case["stats_unit_latency"]["melded"]
        assert m[2] / m[1] > u[2] / u[1]        # utilisation
        du, dm = case["stats_default_latency"]["unmelded"], case["stats_default_latency"]["melded"]
        assert dm[5] < du[5] and dm[6] <= du[6]  # shared / global memory issues
        if case["bucket"] >= 4:
            assert dm[3] < du[3]                 # serialized cycles


@pytest.mark.parametrize("B", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024])
def test_oddeven_restatement_sorts(restatement, B):
    rng = np.random.default_rng(B)
    keys = rng.integers(-(2 ** 31), 2 ** 31, size=B * 16, dtype=np.int64).astype(np.int32)
    want = np.sort(keys.reshape(-1, B), axis=1).reshape(-1)
    restatement.oddeven_sort(keys, B)
    assert (keys == want).all()


SHAPES = [(B, 1) for B in (2, 4, 8, 16, 32, 64, 128, 256, 512, 1024)] + \
         [(B, r) for B in (4, 8, 16, 32, 64, 128, 256, 512) for r in (4, 8, 16) if r <= B and B // r <= 32]


@pytest.mark.gpu
def test_oddeven_gpu_golden():
    gold = load_golden("oddeven_sort.json")
    for case in gold["cases"]:
        B = case["bucket"]
        for kpt in (0, 1, 4, 8, 16):
            if kpt > 1 and (kpt > B or B // kpt > 32):
                continue
            for variant in (0, 1, 2):
                keys = np.array(case["keys"], dtype=np.int32)
                darm.oddeven_sort(keys, B, variant, keys_per_thread=kpt)
                assert keys.tolist() == case["sorted"], (B, kpt, variant)


@pytest.mark.gpu
@pytest.mark.parametrize("bucket,kpt", SHAPES)
def test_oddeven_gpu_vs_restatement(restatement, bucket, kpt):
    import torch

    rng = np.random.default_rng(bucket * 31 + kpt)
    for n in (1 << 17, bucket * 37, bucket):
        for dup in (False, True):
            lo, hi = (-128, 129) if dup else (-(2 ** 31), 2 ** 31)
            keys = rng.integers(lo, hi, size=n, dtype=np.int64).astype(np.int32)
            want = keys.copy()
            restatement.oddeven_sort(want, bucket)
            for variant in (0, 1, 2):
                k = torch.from_numpy(keys.copy()).cuda()
                st = darm.oddeven_sort(k, bucket, variant, keys_per_thread=kpt)
                assert st["keys_per_thread"] == kpt
                assert (k.cpu().numpy() == want).all(), (bucket, kpt, n, dup, variant)


@pytest.mark.gpu
def test_oddeven_gpu_full_size_host_pipeline():
    """2^24 keys, 64-key buckets through the HOST path (pipelined chunks):
    every bucket sorted and a permutation of its input."""
    rng = np.random.default_rng(7)
    keys = rng.integers(-(2 ** 31), 2 ** 31, size=1 << 24, dtype=np.int64).astype(np.int32)
    want = np.sort(keys.reshape(-1, 64), axis=1).reshape(-1)
    for variant in (0, 1, 2):
        k = keys.copy()
        st = darm.oddeven_sort(k, 64, variant)
        assert st["launches"] == 8
        assert (k == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("sort", ["oddeven", "bitonic"])
@pytest.mark.parametrize("bucket", [64, 128, 256])
def test_one_key_shape_many_tiles_per_cta(sort, bucket):
    """One key per thread at 2^22 keys: every CTA walks many 256-key tiles, so
    the shared exchange buffers are reused across tiles (round-2 bench found a
    cross-tile hazard at 2^24 keys that 1-tile-per-CTA sizes never exercised)."""
    import torch

    n = 1 << 22
    g = torch.Generator(device="cuda").manual_seed(bucket)
    keys = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    want = torch.sort(keys.view(-1, bucket), dim=1).values.view(-1)
    fn = darm.oddeven_sort if sort == "oddeven" else darm.bitonic_sort
    for variant in ((0, 1, 2) if sort == "oddeven" else (0, 1, 2, 3)):
        for _ in range(3):
            k = keys.clone()
            fn(k, bucket, variant, keys_per_thread=1, want_stats=False)
            torch.cuda.synchronize()
            assert torch.equal(k, want), (sort, bucket, variant)
