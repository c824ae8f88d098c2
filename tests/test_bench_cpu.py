"""bench.py's CPU-side legs (the cpu_baseline of every per-kernel row and the
ffma2 pattern-roof reader) at small sizes, so a broken baseline surfaces here
and not on the GPU box.  Each returns the cpu_baseline object the bench line
carries: value, unit, cores, kind, sample."""
import os
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402

KEYS = {"value", "unit", "cores", "kind", "sample"}


def _ok(d, unit, kind):
    assert d is not None and KEYS <= set(d), d
    assert d["unit"] == unit and d["kind"] == kind and d["value"] > 0 and d["cores"] >= 1


@pytest.mark.parametrize("net,bucket,kind", [("bitonic", 64, "reference"), ("oddeven", 64, "reference"),
                                             ("bitonic", 1024, "port"), ("oddeven", 256, "port")])
def test_cpu_bucket_sort(net, bucket, kind):
    _ok(bench.cpu_bucket_sort(net, bucket, seconds=0.05), "keys/s", kind)


def test_cpu_corpus_two_parameter_kernel():
    """sb4 takes (h, q): the config-1 split of the GPU rows, compareRuns equal."""
    d = bench.cpu_corpus("sb4", 64)
    _ok(d, "lanes/s", "reference")
    assert d["compare_runs_equal"]


def test_cpu_merge_sort_and_interp():
    _ok(bench.cpu_merge_sort(1 << 14, seconds=0.05), "keys/s", "port")
    _ok(bench.cpu_interp(bench.DIAMOND_IR, 64, seconds=0.05), "warps/s", "reference")


def test_cpu_lud_and_srad_small():
    _ok(bench.cpu_lud(256), "TFLOP/s", "port")
    _ok(bench.cpu_srad(256, 1), "pixel-iterations/s", "port")


def test_pattern_roof_needs_a_gpu():
    """Without a CUDA device the microbenchmark fails and the reader says so."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert bench.ffma2_outer_product_roof() is None
