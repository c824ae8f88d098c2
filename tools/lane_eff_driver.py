"""Launch every kernel family once per form for an ncu lane-efficiency sweep
(run under ncu with the lane-efficiency metrics; see tools/lane_eff.sh)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402

CORPUS = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested", "bitonic"]


def main():
    torch.cuda.set_device(0)
    darm.init()
    nw = 1 << 15
    for k in CORPUS:
        b = darm.make_random_input(k, 32, nw, 1000)
        args = b.args if k == "bitonic" else ([[16]] if len(b.args) == 1 else [[16], [24]])
        for v in ((0, 1) if k == "bitonic" else (0, 1, 2)):   # + the predicated form of the corpus lanes
            g = {n: torch.from_numpy(a.copy()).cuda() for n, a in b.globals.items()}
            sh = {n: torch.from_numpy(a).cuda() for n, a in b.shared.items()} or None
            darm.execute_warps(k, v, 32, args, g, sh, want_stats=False)
    n = 1 << 22
    gen = torch.Generator(device="cuda").manual_seed(3)
    keys = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=gen)
    for sort, forms in ((darm.bitonic_sort, (0, 1, 2, 3)), (darm.oddeven_sort, (0, 1, 2))):
        for kpt in (16, 1):
            for v in forms:
                sort(keys.clone(), 64, v, want_stats=False, keys_per_thread=kpt)
    for v in (0, 1):
        darm.merge_sort(keys[: 1 << 20].clone(), v, want_stats=False)
    for v in (0, 1):
        darm.nqueens(14, 5, v, want_stats=False, mirror=True)
        darm.nqueens(14, 5, v, want_stats=False, mirror=True, paper_shape=True)
    a0 = torch.rand((2048, 2048), generator=gen, device="cuda") + 2048 * torch.eye(2048, device="cuda")
    for v in (0, 1):
        darm.lud(a0.clone(), v, want_stats=False)
    j0 = torch.exp(torch.rand((4096, 4096), generator=gen, device="cuda"))
    for fast in (False, True):
        for v in (0, 1):
            darm.srad(j0.clone(), 2, 0.5, darm.RODINIA_ROI, v, want_stats=False, fast=fast)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
