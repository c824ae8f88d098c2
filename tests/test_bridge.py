"""The reference's acceptance criterion 1 (acceptance.cpp:101-119) through the
reference-side C++ binding include/darm_gpu.hpp: for every positive corpus
kernel, warp sizes {4, 8, 32, 64} and 100 makeRandomInput fixtures, the
reference's compareRuns finds the sm_100a unmelded and melded results equal
to the reference interpreter's; then criteria 5 and 6 (acceptance.cpp:243-310)
with executeWarp replaced by the GPU warp interpreter
(oracle/bridge_test.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

BRIDGE = os.path.join(ROOT, "oracle", "_ref", "bridge_test")


@pytest.mark.gpu
def test_acceptance_c1_on_gpu_through_reference_types():
    if not os.path.exists(BRIDGE):
        pytest.skip("oracle/_ref/bridge_test not built (make -C oracle ref bridge, needs /root/reference)")
    r = subprocess.run([BRIDGE, "100"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "compareRuns verdicts equal" in r.stdout
    # acceptance criteria 5 and 6 with executeWarp replaced by the GPU interpreter
    assert "C5 (GPU interpreter): ok" in r.stdout and "C6 (GPU interpreter): ok" in r.stdout, r.stdout
    # the result oracle itself (testing::oracleCompare) on the GPU, incl. a mutated kernel it must catch
    assert "GPU oracle (oracleCompare on executeWarpsIR): ok" in r.stdout, r.stdout


GPU_BENCH = os.path.join(ROOT, "oracle", "_ref", "darm_gpu_bench")
# the keys of the reference's `darm bench` JSON rows (tools/darm_cli.cpp:343-358)
REFERENCE_ROW_KEYS = {"kernel", "mode", "threshold", "rejected", "melded", "melds", "converged", "mpScores",
                      "oracleOk", "oracleDiff", "serializedBefore", "serializedAfter",
                      "serializedReductionPercent", "utilizationBefore", "utilizationAfter"}
GPU_ROW_KEYS = {"gpuOracleOk", "gpuOracleDiff", "gpuLanes", "gpuUnmeldedUs", "gpuMeldedUs", "gpuSpeedup",
                "gpuSimEqual", "cpuSimMs", "gpuSimMs"}


def _gpu_bench(args, tmp_path):
    import json

    if not os.path.exists(GPU_BENCH):
        pytest.skip("oracle/_ref/darm_gpu_bench not built (make -C oracle gpubench, needs /root/reference)")
    out = tmp_path / "rows.json"
    r = subprocess.run([GPU_BENCH, *args, "--json", str(out)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(out.read_text()), r.stdout


def test_stats_wire_format_reference_rows(tmp_path):
    """The bench rows carry the reference's keys (plus the gpu* columns, null
    without a GPU) and the reference simulator's numbers for every kernel."""
    rows, table = _gpu_bench(["--no-gpu", "--fixtures", "4"], tmp_path)
    assert [r["kernel"] for r in rows] == ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested",
                                           "bitonic"]
    for r in rows:
        assert REFERENCE_ROW_KEYS | GPU_ROW_KEYS == set(r)
        assert r["oracleOk"] and r["melded"] and r["serializedAfter"] < r["serializedBefore"]
        assert r["gpuUnmeldedUs"] is None
    assert "ser.pre" in table and "gpu.x" in table


@pytest.mark.gpu
def test_stats_wire_format_gpu_rows(tmp_path):
    rows, _ = _gpu_bench(["--fixtures", "20", "--gpu-warps", "32768"], tmp_path)
    for r in rows:
        assert r["gpuOracleOk"], (r["kernel"], r["gpuOracleDiff"])
        assert r["gpuSimEqual"], r["kernel"]      # the simulator statistics, computed on the GPU
        assert r["gpuLanes"] == 32 * 32768
        assert r["gpuUnmeldedUs"] > 0 and r["gpuMeldedUs"] > 0
