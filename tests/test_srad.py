"""SRAD (no reference code): the CPU restatement, the
row-tiled multi-rank driver (gloo, world 2/3, on CPU with numpy tile kernels)
and — on the GPU — both forms bit-exact against the restatement, the tiled
path against the single-GPU path, and the BASELINE config 5 size."""
import os
import socket
import threading

import numpy as np
import pytest
import torch

import paper_2107_05681_b200 as darm
from paper_2107_05681_b200.srad_tiles import SradTiles, split_rows
from srad_numpy import NumpyTileKernels

ROI = (0, 127, 0, 127)


def image(rows, cols, seed=0):
    rng = np.random.default_rng(seed)
    return np.exp(rng.random((rows, cols), dtype=np.float32)).astype(np.float32)


def test_restatement_max_principle(restatement):
    j = image(200, 300)
    lo, hi = j.min(), j.max()
    restatement.srad(j, 10, 0.5, ROI)
    assert j.min() >= lo * (1 - 1e-6) and j.max() <= hi * (1 + 1e-6)
    assert np.isfinite(j).all()


def test_restatement_threads_do_not_change_bits(restatement):
    a = image(130, 97, 1)
    b = a.copy()
    restatement.srad(a, 5, 0.5, (3, 60, 5, 90), threads=1)
    restatement.srad(b, 5, 0.5, (3, 60, 5, 90), threads=5)
    assert (a.view(np.int32) == b.view(np.int32)).all()


@pytest.mark.parametrize("rows,cols,roi", [(64, 70, ROI[:1] + (40, 0, 69)), (130, 97, (3, 60, 5, 90))])
def test_numpy_tile_kernels_match_restatement(restatement, rows, cols, roi):
    j = image(rows, cols, 2)
    want = j.copy()
    restatement.srad(want, 4, 0.5, roi)
    t = SradTiles(rows, cols, 0.5, roi, kernels=NumpyTileKernels())
    t.load(torch.from_numpy(j))
    t.run(4)
    assert (t.gather().numpy().view(np.int32) == want.view(np.int32)).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, rows, cols, roi, iters, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = SradTiles(rows, cols, 0.5, roi, kernels=NumpyTileKernels(), dist=dist)
        t.load(torch.from_numpy(image(rows, cols, 3)))
        t.run(iters)
        full = t.gather()
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_tiled_halo_exchange_gloo(restatement, world):
    """world_size 2/3 gloo processes: halos + ROI all-reduce reproduce the
    single-image restatement bit for bit (ROI rows spread over ranks)."""
    import torch.multiprocessing as mp

    rows, cols, roi, iters = 41, 67, (5, 30, 3, 60), 3
    want = image(rows, cols, 3)
    restatement.srad(want, iters, 0.5, roi)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, rows, cols, roi, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert (got.view(np.int32) == want.view(np.int32)).all()


def test_split_rows():
    assert split_rows(10, 3) == [(0, 4), (4, 3), (7, 3)]
    with pytest.raises(darm.DarmUserError):
        split_rows(3, 2)


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("rows,cols,iters,roi", [(256, 256, 20, ROI), (513, 377, 7, (10, 200, 31, 300)),
                                                  (64, 2, 3, (0, 63, 0, 1)), (2049, 1000, 4, ROI)])
def test_gpu_bit_exact_vs_restatement(restatement, variant, rows, cols, iters, roi):
    j = image(rows, cols, rows)
    want = j.copy()
    restatement.srad(want, iters, 0.5, roi)
    darm.srad(j, iters, 0.5, roi, variant)
    assert (j.view(np.int32) == want.view(np.int32)).all(), np.abs(j - want).max()


class _ThreadDist:
    """In-process stand-in for torch.distributed (threads = ranks) so the
    tiled path runs with the real GPU kernels on one GPU."""

    P2POp = None

    def __init__(self, world):
        self.world = world
        self.box = {}
        self.cv = threading.Condition()
        self.barrier = threading.Barrier(world)
        self.red = [None] * world
        self.local = threading.local()

        class Op:
            def __init__(op, fn, t, peer):
                op.fn, op.t, op.peer = fn, t, peer

        self.P2POp = Op
        self.ReduceOp = type("R", (), {"SUM": "sum"})

    def get_world_size(self):
        return self.world

    def get_backend(self):
        return "nccl"   # device tensors straight through, like NCCL

    def get_rank(self):
        return self.local.rank

    def isend(self):
        pass

    def irecv(self):
        pass

    def batch_isend_irecv(self, ops):
        me = self.local.rank
        with self.cv:
            for op in ops:
                if op.fn == self.isend:
                    self.box[(me, op.peer)] = op.t.clone()
            self.cv.notify_all()
        for op in ops:
            if op.fn == self.irecv:
                with self.cv:
                    self.cv.wait_for(lambda: (op.peer, me) in self.box)
                    op.t.copy_(self.box.pop((op.peer, me)))
        return []

    def all_reduce(self, t, op=None):
        me = self.local.rank
        self.red[me] = t.clone()
        self.barrier.wait()
        total = self.red[0].clone()
        for k in range(1, self.world):
            total += self.red[k]
        self.barrier.wait()
        t.copy_(total)

    def send(self, t, dst):
        with self.cv:
            self.box[(self.local.rank, dst)] = t.clone()
            self.cv.notify_all()

    def recv(self, t, src):
        with self.cv:
            self.cv.wait_for(lambda: (src, self.local.rank) in self.box)
            t.copy_(self.box.pop((src, self.local.rank)))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 3, 4])
def test_gpu_tiled_equals_single(world):
    rows, cols, iters, roi = 600, 333, 6, (100, 250, 0, 200)   # ROI rows straddle tiles
    j = image(rows, cols, 9)
    want = j.copy()
    darm.srad(want, iters, 0.5, roi, 1)
    dist = _ThreadDist(world)
    out = {}

    def run(rank):
        dist.local.rank = rank
        torch.cuda.set_device(0)
        t = SradTiles(rows, cols, 0.5, roi, dist=dist, device=torch.device("cuda", 0))
        t.load(torch.from_numpy(j).cuda())
        for _ in range(iters):
            t.step()
            torch.cuda.synchronize()
        full = t.gather()
        if rank == 0:
            out["img"] = full.cpu().numpy()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert (out["img"].view(np.int32) == want.view(np.int32)).all()


@pytest.mark.gpu
def test_gpu_config5_16384(restatement):
    """BASELINE config 5: 16384^2 fp32, 100 iterations.  Both forms agree bit
    for bit, the max principle holds, and one iteration equals the CPU
    restatement bit for bit (within 1e-5 relative is asserted too)."""
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(5)
    j0 = torch.exp(torch.rand((n, n), generator=g, device="cuda"))
    res = {}
    for v in (0, 1):
        j = j0.clone()
        darm.srad(j, 100, 0.5, ROI, v)
        torch.cuda.synchronize()
        res[v] = j
    assert torch.equal(res[0], res[1])
    assert float(res[1].min()) >= float(j0.min()) * (1 - 1e-6)
    assert float(res[1].max()) <= float(j0.max()) * (1 + 1e-6)
    one = j0.clone()
    darm.srad(one, 1, 0.5, ROI, 1)
    want = j0.cpu().numpy()
    restatement.srad(want, 1, 0.5, ROI)
    got = one.cpu().numpy()
    assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-5
    assert (got.view(np.int32) == want.view(np.int32)).all()


@pytest.mark.gpu
def test_gpu_config5_16384_100_iterations_vs_restatement(restatement):
    """BASELINE config 5 at full size and full length: 16384^2 x 100 on the GPU
    (melded, IEEE) equals the CPU restatement run for all 100 iterations on
    every host thread, bit for bit; the fast-math form stays within the north
    star's 1e-5 relative of it."""
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(6)
    j0 = torch.exp(torch.rand((n, n), generator=g, device="cuda"))
    want = j0.cpu().numpy()
    restatement.srad(want, 100, 0.5, ROI, threads=os.cpu_count() or 1)
    j = j0.clone()
    darm.srad(j, 100, 0.5, ROI, 1)
    got = j.cpu().numpy()
    assert (got.view(np.int32) == want.view(np.int32)).all(), float(np.max(np.abs(got - want) / np.abs(want)))
    f = j0.clone()
    darm.srad(f, 100, 0.5, ROI, 1, fast=True)
    rel = float(np.max(np.abs(f.cpu().numpy() - want) / np.abs(want)))
    assert rel <= 1e-5, rel


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("rows,cols,iters,roi", [(256, 256, 100, ROI), (513, 377, 30, (10, 200, 31, 300)),
                                                  (2049, 1000, 20, ROI)])
def test_gpu_fast_math_within_tolerance(restatement, variant, rows, cols, iters, roi):
    """DARM_FAST_MATH: the north star's 1e-5 relative tolerance against the
    IEEE restatement, after up to 100 iterations; the two forms agree bit for
    bit with each other."""
    j0 = image(rows, cols, rows + 1)
    want = j0.copy()
    restatement.srad(want, iters, 0.5, roi)
    j = j0.copy()
    darm.srad(j, iters, 0.5, roi, variant, fast=True)
    rel = np.max(np.abs(j - want) / np.abs(want))
    assert rel <= 1e-5, rel
    other = j0.copy()
    darm.srad(other, iters, 0.5, roi, 1 - variant, fast=True)
    assert (other.view(np.int32) == j.view(np.int32)).all()


@pytest.mark.gpu
def test_gpu_fast_math_config5(restatement):
    """16384^2: 100 fast iterations stay within 1e-5 relative of 100 IEEE
    iterations on the GPU (the IEEE path is bit-exact to the restatement)."""
    n = 16384
    g = torch.Generator(device="cuda").manual_seed(5)
    j0 = torch.exp(torch.rand((n, n), generator=g, device="cuda"))
    a, b = j0.clone(), j0.clone()
    darm.srad(a, 100, 0.5, ROI, 1)
    darm.srad(b, 100, 0.5, ROI, 1, fast=True)
    torch.cuda.synchronize()
    rel = float(((a - b).abs() / a.abs()).max())
    assert rel <= 1e-5, rel
