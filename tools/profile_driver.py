"""Launch the hot kernels once per form for ncu captures (run under gpurun).

    ncu ... python tools/profile_driver.py bitonic   # 2^24 keys, B=64, unmelded then melded
    ncu ... python tools/profile_driver.py sb1       # 2^20 lanes, n=16, unmelded then melded
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402


def main(which, bucket=64):
    torch.cuda.set_device(0)
    darm.init()
    if which == "lud":
        n = bucket if bucket > 64 else 8192
        g = torch.Generator(device="cuda").manual_seed(4)
        a0 = torch.rand((n, n), generator=g, device="cuda") + n * torch.eye(n, device="cuda")
        for v in (darm.UNMELDED, darm.MELDED):
            a = a0.clone()
            darm.lud(a, v, want_stats=False)
        torch.cuda.synchronize()
        return
    if which == "srad":
        n = 16384
        g = torch.Generator(device="cuda").manual_seed(5)
        j0 = torch.exp(torch.rand((n, n), generator=g, device="cuda"))
        for fast in (False, True):       # one sweep per form: IEEE unmelded, melded, then fast
            for v in (darm.UNMELDED, darm.MELDED):
                j = j0.clone()
                darm.srad(j, 1, 0.5, darm.RODINIA_ROI, v, want_stats=False, fast=fast)
        torch.cuda.synchronize()
        return
    if which == "interp":   # bench.py's interpreter row: the diamond IR, 32,768 warps of 32 lanes
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from bench import DIAMOND_IR

        prog = darm.Program(DIAMOND_IR)
        nwi = 1 << 15
        g = torch.Generator(device="cuda").manual_seed(3)
        gi = torch.randint(-128, 129, (nwi, prog.global_words), dtype=torch.int32, device="cuda", generator=g)
        prog.execute_warps(32, np.full((1, 1), 16, np.int32), gi, n_warps=nwi)
        torch.cuda.synchronize()
        return
    if which == "nqueens_step":   # the paper-shaped encoding, the bench's launch
        for v in (darm.UNMELDED, darm.MELDED):
            assert darm.nqueens(16, 7, v, want_stats=False, mirror=True, paper_shape=True)[0] == 14772512
        return
    if which == "nqueens":
        for v in (darm.UNMELDED, darm.MELDED):   # the bench's launch: 7-row prefixes, mirror symmetry
            assert darm.nqueens(16, 7, v, want_stats=False, mirror=True)[0] == 14772512
        return
    if which == "merge":
        n = bucket if bucket > 64 else 1 << 24
        g = torch.Generator(device="cuda").manual_seed(9)
        pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        for v in (darm.UNMELDED, darm.MELDED):
            k = pristine.clone()
            darm.merge_sort(k, v, want_stats=False)
        torch.cuda.synchronize()
        return
    if which == "oddeven":
        n = 1 << 24
        g = torch.Generator(device="cuda").manual_seed(1234)
        pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        for kpt in (0, 1):
            for v in (darm.UNMELDED, darm.MELDED):
                k = pristine.clone()
                darm.oddeven_sort(k, bucket, v, want_stats=False, keys_per_thread=kpt)
        torch.cuda.synchronize()
        return
    if which == "bitonic":
        n = 1 << 24
        g = torch.Generator(device="cuda").manual_seed(1234)
        pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        kpts = (0, 1) if bucket <= 1024 else (0,)
        for kpt in kpts:       # register-blocked (auto: 16 keys per thread), then one key per thread
            for v in (darm.UNMELDED, darm.MELDED, darm.PREDICATED, darm.MELDED_LITERAL):
                k = pristine.clone()
                darm.bitonic_sort(k, bucket, v, want_stats=False, keys_per_thread=kpt)
        torch.cuda.synchronize()
    else:
        nw = 1 << 15
        b = darm.make_random_input(which, 32, nw, 1000)
        args = [[16]] if len(darm.kernel_info(which)["params"]) == 1 else [[16], [24]]
        for v in (darm.UNMELDED, darm.MELDED, darm.PREDICATED):
            g = {n: torch.from_numpy(a.copy()).cuda() for n, a in b.globals.items()}
            sh = {n: torch.from_numpy(a).cuda() for n, a in b.shared.items()} or None
            darm.execute_warps(which, v, 32, args if which != "bitonic" else b.args, g, sh, want_stats=False)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 64)
