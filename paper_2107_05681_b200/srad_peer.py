"""Peer-memory row-tiled SRAD across GPUs (BASELINE config 5, the product path).

One process per GPU, one :class:`SradPeerTiles` per rank, over the C-ABI's
``darm_gpu_srad_group_*`` (include/darm_gpu.h).  torch.distributed is only the
plumbing that hands every rank the others' 128-byte handles (CUDA IPC memory
handles) and gathers the image at the end; the per-iteration exchange needs no
collective: each rank's GPU reads its halo rows and the ROI partial sums
straight out of its neighbours' memory over NVLink / NVSwitch, the ranks keep
phase with flags in device memory, and all iterations of a run are one CUDA
graph (halo pull on a side stream beside the interior rows, then the edge
rows).  Results are bit-identical to the single-GPU ``darm.srad``.

Ranks in one process (tests on one GPU) share pointers directly; ranks in
different processes open each other's memory by CUDA IPC.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import paper_2107_05681_b200 as darm

HANDLE_BYTES = 128


class SradPeerTiles:
    """This rank's tile of a peer-memory row-tiled SRAD run."""

    def __init__(self, rows: int, cols: int, lam: float = 0.5, roi: Sequence[int] = darm.RODINIA_ROI,
                 dist=None, variant=darm.MELDED, fast: bool = False, rank: Optional[int] = None,
                 world: Optional[int] = None, exchange=None):
        import torch

        self.torch = torch
        self.dist = dist
        self.world = world if world is not None else (dist.get_world_size() if dist else 1)
        self.rank = rank if rank is not None else (dist.get_rank() if dist else 0)
        self.rows, self.cols = int(rows), int(cols)
        if isinstance(variant, str):
            variant = darm.VARIANTS[variant]
        if fast:
            variant |= darm.FAST_MATH
        L = darm.lib()
        self._g = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(HANDLE_BYTES)
        err = ctypes.create_string_buffer(512)
        self._roi = darm._roi_arr(roi)
        darm._check(L.darm_gpu_srad_group_create(int(variant), self.rows, self.cols, float(lam), self._roi,
                                                 self.rank, self.world, ctypes.byref(self._g), handle, err, 512), err)
        mine = bytes(handle.raw)
        if exchange is not None:          # in-process ranks (tests): a callable all-gather
            handles = exchange(self.rank, mine)
        elif self.world > 1:
            handles = [None] * self.world
            dist.all_gather_object(handles, mine)
        else:
            handles = [mine]
        blob = ctypes.create_string_buffer(b"".join(handles), HANDLE_BYTES * self.world)
        darm._check(L.darm_gpu_srad_group_connect(self._g, blob, err, 512), err)
        r0, n = ctypes.c_int64(), ctypes.c_int64()
        L.darm_gpu_srad_group_rows(self._g, ctypes.byref(r0), ctypes.byref(n))
        self.r0, self.n = int(r0.value), int(n.value)
        if exchange is None and self.world > 1:
            dist.barrier()

    def _stream(self, stream):
        return stream if stream is not None else self.torch.cuda.current_stream().cuda_stream

    def load(self, image, stream=None) -> None:
        """This rank's rows of the full image (rows x cols), or the rows themselves."""
        t = image[self.r0:self.r0 + self.n] if image.shape[0] == self.rows else image
        err = ctypes.create_string_buffer(512)
        if darm._is_torch_cuda(t):
            t = t.contiguous()
            self._keep = t
            darm._check(darm.lib().darm_gpu_srad_group_load(self._g, ctypes.c_void_p(t.data_ptr()), 1,
                                                            ctypes.c_void_p(self._stream(stream)), err, 512), err)
        else:
            import numpy as np

            a = np.ascontiguousarray(t, dtype=np.float32)
            darm._check(darm.lib().darm_gpu_srad_group_load(self._g, ctypes.c_void_p(a.ctypes.data), 0,
                                                            ctypes.c_void_p(self._stream(stream)), err, 512), err)

    def run(self, iters: int, stream=None, want_stats: bool = False):
        st = darm.Stats()
        err = ctypes.create_string_buffer(512)
        darm._check(darm.lib().darm_gpu_srad_group_run(self._g, int(iters), ctypes.c_void_p(self._stream(stream)),
                                                       ctypes.byref(st) if want_stats else None, err, 512), err)
        return st.as_dict() if want_stats else None

    def tile(self, stream=None):
        """This rank's rows (n x cols) as a CUDA tensor (synchronises; raises if a peer timed out)."""
        out = self.torch.empty((self.n, self.cols), dtype=self.torch.float32, device="cuda")
        err = ctypes.create_string_buffer(512)
        darm._check(darm.lib().darm_gpu_srad_group_read(self._g, ctypes.c_void_p(out.data_ptr()), 1,
                                                        ctypes.c_void_p(self._stream(stream)), err, 512), err)
        return out

    def gather(self):
        """The full image on rank 0 (None elsewhere); torch.distributed point-to-point."""
        own = self.tile()
        if self.world == 1:
            return own
        from paper_2107_05681_b200.srad_tiles import split_rows

        torch = self.torch
        stage = self.dist.get_backend() == "gloo"
        dev = torch.device("cpu") if stage else own.device
        if self.rank == 0:
            out = [own.to(dev)]
            for k, (_, n) in list(enumerate(split_rows(self.rows, self.world)))[1:]:
                part = torch.empty((n, self.cols), dtype=torch.float32, device=dev)
                self.dist.recv(part, src=k)
                out.append(part)
            return torch.cat(out, dim=0).to(own.device)
        self.dist.send(own.to(dev), dst=0)
        return None

    def close(self) -> None:
        if getattr(self, "_g", None) and self._g.value:
            darm.lib().darm_gpu_srad_group_free(self._g)
            self._g = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
