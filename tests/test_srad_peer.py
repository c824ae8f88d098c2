"""Peer-memory row-tiled SRAD (darm_gpu_srad_group_*, paper_2107_05681_b200.srad_peer):
the multi-GPU product path.  Halos and ROI partials are read from the
neighbours' memory, phases are kept with device flags, the iteration loop is
one CUDA graph — and the gathered image must equal the single-GPU darm.srad bit
for bit (IEEE and fast-math, both forms).

Only one GPU is available to this build: ranks run as threads of one process
on cuda:0 (pointers shared directly), and as two processes on cuda:0 (the CUDA
IPC path an 8-GPU run takes, handles exchanged over gloo).  On one GPU the
ranks' spinning phase waits share the device's hardware queues, which can
serialise a waiter in front of the work it waits for — a hazard an 8-GPU run
(one rank per GPU) does not have.  Threads of one process share one context,
and with the streams earlier tests leave behind two ranks' streams can alias
onto one hardware queue (a round-2 suite run timed out that way), so every
multi-rank thread case advances in host lockstep (one-iteration graphs, a
host barrier between iterations).  The free-running multi-iteration graph is
exercised by the two-process case (separate contexts time-slice, so a waiter
cannot hold back the rank it waits for indefinitely).
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch

import paper_2107_05681_b200 as darm

ROI = (0, 127, 0, 127)


def image(rows, cols, seed=0):
    rng = np.random.default_rng(seed)
    return np.exp(rng.random((rows, cols), dtype=np.float32)).astype(np.float32)


def run_threads(world, rows, cols, iters, roi, variant, fast, runs=1, lockstep=False):
    from paper_2107_05681_b200.srad_peer import SradPeerTiles

    img = torch.from_numpy(image(rows, cols, rows + cols)).cuda()
    box, bar = [None] * world, threading.Barrier(world)
    parts, errors = [None] * world, []

    def exchange(rank, h):
        box[rank] = h
        bar.wait()
        return list(box)

    def rank_main(rank):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                t = SradPeerTiles(rows, cols, 0.5, roi, variant=variant, fast=fast, rank=rank, world=world,
                                  exchange=exchange)
                for _ in range(runs):
                    t.load(img)
                    if lockstep:
                        s.synchronize()
                        bar.wait()
                        for _ in range(iters):
                            t.run(1)
                            s.synchronize()
                            bar.wait()
                    else:
                        t.run(iters)
                parts[rank] = (t.r0, t.tile().cpu().numpy())
                bar.wait()   # nobody frees its memory while a peer may still read it
                t.close()
        except Exception as e:   # pragma: no cover - reported below
            errors.append(repr(e))
            bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=300)
    assert not errors, errors
    parts.sort(key=lambda p: p[0])
    return np.concatenate([p[1] for p in parts])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("variant,fast", [(0, False), (1, False), (1, True)])
def test_peer_tiles_equal_single_gpu(world, variant, fast):
    rows, cols, iters, roi = 601, 333, 7, (100, 250, 0, 200)   # ROI rows straddle the tiles
    want = image(rows, cols, rows + cols)
    darm.srad(want, iters, 0.5, roi, variant, fast=fast)
    got = run_threads(world, rows, cols, iters, roi, variant, fast, lockstep=world > 1)
    assert (got.view(np.int32) == want.view(np.int32)).all()


@pytest.mark.gpu
def test_peer_tiles_graph_reused_across_runs():
    """Two load+run rounds through the same cached graph (device-resident phase
    counters, nothing baked in): the second round reproduces the first."""
    rows, cols, iters = 300, 260, 5
    want = image(rows, cols, rows + cols)
    darm.srad(want, iters, 0.5, ROI, 1)
    got = run_threads(2, rows, cols, iters, ROI, 1, False, runs=2, lockstep=True)
    assert (got.view(np.int32) == want.view(np.int32)).all()


@pytest.mark.gpu
def test_peer_tiles_thin_tiles():
    """Tiles of 2-3 rows (no interior rows: every row is an edge row)."""
    rows, cols, iters = 9, 130, 4
    want = image(rows, cols, rows + cols)
    darm.srad(want, iters, 0.5, (0, 8, 0, 129), 1)
    got = run_threads(4, rows, cols, iters, (0, 8, 0, 129), 1, False, lockstep=True)
    assert (got.view(np.int32) == want.view(np.int32)).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), DARM_PEER_TIMEOUT_S="60")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2107_05681_b200.srad_peer import SradPeerTiles

        torch.cuda.set_device(0)
        rows, cols, iters = 257, 300, 6
        img = image(rows, cols, 11)
        t = SradPeerTiles(rows, cols, 0.5, ROI, dist=dist, variant=1)
        t.load(torch.from_numpy(img).cuda())
        t.run(iters)
        full = t.gather()
        dist.barrier()
        t.close()
        if rank == 0:
            want = img.copy()
            darm.srad(want, iters, 0.5, ROI, 1)
            q.put(bool((full.cpu().numpy().view(np.int32) == want.view(np.int32)).all()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_peer_tiles_two_processes_ipc():
    """Two processes on cuda:0: handles over gloo, tiles opened by CUDA IPC."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
