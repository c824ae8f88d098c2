"""bench.py's multi-rank path.

`bench.py --gpus 2` must launch two ranks itself (torch.distributed.run on
127.0.0.1), each rank one process, and print n_gpus == 2 with the work of both
ranks in `value` / `global_batch`.  Only one GPU is available to this build, so
both ranks run on cuda:0 and talk over gloo (DARM_DIST_BACKEND=gloo: NCCL
refuses two ranks on one device) — the rank logic, the sharding and the
exchange steps are the ones an 8-GPU NCCL run executes.

Bit-exactness against one GPU:
  * bitonic: every rank checks its sorted keys against torch.sort inside bench.py;
  * N-Queens: the prefix shards of both ranks sum to Q(16) = 14,772,512 (asserted in bench.py);
  * SRAD: the row-tiled image gathered on rank 0 hashes to the same bytes as
    the single-GPU run, through both transports (peer-memory tiles over CUDA
    IPC, and torch.distributed halos + ROI all-reduce).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(gpus, *extra, timeout=900):
    env = dict(os.environ, DARM_DIST_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--steps", "3", "--warmup", "3",
           "--keys", str(1 << 20), "--no-cpu-baseline", *extra]
    p = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_two_ranks_match_one_gpu():
    args = ("--kernels", "nqueens16,srad", "--srad-size", "1030", "--srad-iters", "7")
    one = run_bench(1, *args)
    two = run_bench(2, *args)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["config"]["global_batch"] == 2 * (1 << 20)
    assert two["config"]["parallelism"].startswith("dp2")
    nq = two["per_kernel"]["nqueens16"]
    assert nq["n_gpus"] == 2 and nq["melded_solutions"] == nq["unmelded_solutions"] == 14772512
    for key in ("srad1030x7", "srad1030x7_fast_math"):
        r1, r2 = one["per_kernel"][key], two["per_kernel"][key]
        assert r2["n_gpus"] == 2
        for form in ("unmelded", "melded"):
            assert r1[form + "_result_sha16"] == r2[form + "_result_sha16"], (key, form)
        # the torch.distributed transport (P2P halos + ROI all-reduce) gives the same bits
        assert r2["melded_torch_dist_result_sha16"] == r1["melded_result_sha16"], key


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--no-per-kernel",
                        "--no-cpu-baseline"], env=env, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE=1" in (p.stdout + p.stderr)
