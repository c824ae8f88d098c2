"""Row-tiled SRAD across GPUs (BASELINE config 5: 16384^2, 100 iterations).

One process per GPU (torch.distributed); rank k owns image rows
[r0_k, r0_k + rows_k).  Each tile buffer holds its rows at local rows
1..rows_k plus one halo row above (local 0) and two below (local rows_k+1,
rows_k+2) — the fused sweep kernel needs J(i-1) .. J(i+2); rows are
`darm.srad_pitch(cols)` floats (16-byte rows).  Per iteration:

  1. all-reduce (sum) of the ROI partial-sum buffer: every entry is written by
     exactly one rank (the owner of that ROI row), so the sum is exact and
     every rank gets the same q0sqr;
  2. the halo exchange (the path's one real exchange step) is POSTED: rank k
     sends its last own row down to k+1 and its first two own rows up to k-1
     (torch.distributed P2P: NCCL over NVLink on GPUs, gloo in CPU tests);
  3. while it is in flight, the interior rows (which read no halo row) run:
     darm_gpu_srad_tile_step(part=DARM_SRAD_INTERIOR_ROWS) — q0sqr + the fused
     sweep J -> J' on rows 2 .. rows_k-2;
  4. the exchange is waited for (NCCL: the compute stream waits on the
     communication stream, no host sync) and the edge rows run
     (part=DARM_SRAD_EDGE_ROWS).

This is the NCCL/torch.distributed transport.  The peer-memory transport
(paper_2107_05681_b200.srad_peer: ranks read their halos straight from the
neighbours' tiles over NVLink, the whole iteration loop one CUDA graph) is
the B200 product path; this one is its baseline and the CPU-testable spec.

The tile-level kernels are injected (``kernels``), so the exchange logic is
exercised on CPU with the oracle's tile kernels in tests/test_srad.py; the
product default is :class:`GpuTileKernels` (libdarm_gpu.so, no fallback).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import paper_2107_05681_b200 as darm


def split_rows(rows: int, world: int) -> List[Tuple[int, int]]:
    """(r0, n) for every rank; every tile has at least 2 rows."""
    base, extra = divmod(rows, world)
    out, r0 = [], 0
    for k in range(world):
        n = base + (1 if k < extra else 0)
        out.append((r0, n))
        r0 += n
    if any(n < 2 for _, n in out):
        raise darm.DarmUserError("every rank needs at least 2 image rows")
    return out


class GpuTileKernels:
    """Tile kernels through the C-ABI (device tensors on the current stream)."""

    def __init__(self, variant, stream=None):
        self.variant = variant
        self.stream = stream

    def roi(self, tile, cols, tile_rows, r0, rows, roi, roi_out):
        darm.srad_tile_roi(tile, cols, tile_rows, r0, rows, roi, roi_out, self.stream)

    def step(self, tin, tout, cols, tile_rows, r0, rows, lam, roi, roi_in, roi_out, q0, part=0):
        darm.srad_tile_step(self.variant, tin, tout, cols, tile_rows, r0, rows, lam, roi, roi_in, roi_out, q0,
                            self.stream, part)


class SradTiles:
    """This rank's tile of a row-tiled SRAD run."""

    def __init__(self, rows: int, cols: int, lam: float = 0.5, roi: Sequence[int] = darm.RODINIA_ROI,
                 kernels=None, dist=None, device=None, variant=darm.MELDED):
        import torch

        self.torch = torch
        self.dist = dist
        self.world = dist.get_world_size() if dist else 1
        self.rank = dist.get_rank() if dist else 0
        self.rows, self.cols, self.lam, self.roi = rows, cols, float(lam), tuple(int(x) for x in roi)
        self.r0, self.n = split_rows(rows, self.world)[self.rank]
        self.device = device if device is not None else torch.device("cpu")
        self.kernels = kernels if kernels is not None else GpuTileKernels(variant)
        self.pitch = darm.srad_pitch(cols)
        shape = (self.n + 3, self.pitch)
        self.tin = torch.zeros(shape, dtype=torch.float32, device=self.device)
        self.tout = torch.zeros(shape, dtype=torch.float32, device=self.device)
        words = darm.srad_roi_words(cols, self.roi)
        self.roi_in = torch.zeros(words, dtype=torch.float64, device=self.device)
        self.roi_out = torch.zeros(words, dtype=torch.float64, device=self.device)
        self.q0 = torch.zeros(1, dtype=torch.float32, device=self.device)

    # ---------------------------------------------------------------- data
    def load(self, image) -> None:
        """Copy this rank's rows of the full image (or the tile rows) in."""
        if image.shape[0] == self.rows:
            self.tin[1:self.n + 1, :self.cols].copy_(image[self.r0:self.r0 + self.n])
        else:
            self.tin[1:self.n + 1, :self.cols].copy_(image)
        self.kernels.roi(self.tin, self.cols, self.n, self.r0, self.rows, self.roi, self.roi_in)

    def tile(self):
        return self.tin[1:self.n + 1, :self.cols]

    # ---------------------------------------------------------------- exchange
    def post_halos(self):
        """Start the halo exchange; returns a finish() that lands the halo rows
        (NCCL: recv straight into the tile rows, the compute stream waits on
        the communication stream; gloo: host-staged, copied in on finish)."""
        if self.world == 1:
            return lambda: None
        d = self.dist
        # gloo moves host buffers only (NCCL moves device memory directly)
        stage = self.device.type == "cuda" and d.get_backend() == "gloo"
        to_wire = (lambda t: t.cpu()) if stage else (lambda t: t.contiguous())  # noqa: E731
        ops = []
        up, down = self.rank - 1, self.rank + 1
        top = bottom = None
        if up >= 0:
            top = self.halo_top.cpu() if stage else self.tin[0:1]
            ops.append(d.P2POp(d.isend, to_wire(self.tin[1:3]), up))
            ops.append(d.P2POp(d.irecv, top, up))
        if down < self.world:
            bottom = self.halo_bottom.cpu() if stage else self.tin[self.n + 1:self.n + 3]
            ops.append(d.P2POp(d.isend, to_wire(self.tin[self.n:self.n + 1]), down))
            ops.append(d.P2POp(d.irecv, bottom, down))
        reqs = d.batch_isend_irecv(ops)

        def finish():
            for req in reqs:
                req.wait()
            if stage:
                if up >= 0:
                    self.tin[0:1].copy_(top)
                if down < self.world:
                    self.tin[self.n + 1:self.n + 3].copy_(bottom)
        return finish

    def exchange_halos(self) -> None:
        self.post_halos()()

    @property
    def halo_top(self):
        if not hasattr(self, "_ht"):
            self._ht = self.torch.empty((1, self.pitch), dtype=self.torch.float32, device=self.device)
        return self._ht

    @property
    def halo_bottom(self):
        if not hasattr(self, "_hb"):
            self._hb = self.torch.empty((2, self.pitch), dtype=self.torch.float32, device=self.device)
        return self._hb

    # ---------------------------------------------------------------- iterate
    def step(self) -> None:
        args = (self.tin, self.tout, self.cols, self.n, self.r0, self.rows, self.lam, self.roi, self.roi_in,
                self.roi_out, self.q0)
        if self.world == 1:
            self.kernels.step(*args, part=darm.SRAD_ALL_ROWS)
        else:
            self.dist.all_reduce(self.roi_in, op=self.dist.ReduceOp.SUM)
            finish = self.post_halos()
            self.kernels.step(*args, part=darm.SRAD_INTERIOR_ROWS)   # overlaps the halo transfer
            finish()
            self.kernels.step(*args, part=darm.SRAD_EDGE_ROWS)
        self.tin, self.tout = self.tout, self.tin
        self.roi_in, self.roi_out = self.roi_out, self.roi_in

    def run(self, iters: int) -> None:
        for _ in range(iters):
            self.step()

    def gather(self) -> Optional[object]:
        """The full image on rank 0 (None elsewhere)."""
        torch = self.torch
        if self.world == 1:
            return self.tile().clone()
        stage = self.device.type == "cuda" and self.dist.get_backend() == "gloo"
        dev = torch.device("cpu") if stage else self.device
        parts = [torch.empty((n, self.cols), dtype=torch.float32, device=dev)
                 for _, n in split_rows(self.rows, self.world)]
        own = self.tile().contiguous().to(dev)
        if self.rank == 0:
            out = [own.clone()]
            for k in range(1, self.world):
                self.dist.recv(parts[k], src=k)
                out.append(parts[k])
            return torch.cat(out, dim=0).to(self.device)
        self.dist.send(own, dst=0)
        return None
