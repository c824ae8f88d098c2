"""GPU executeWarp (darm_gpu_program_execute) vs the reference interpreter on the
host cores, for makeRandomInput batches of corpus kernels (run under gpurun)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2107_05681_b200 as darm  # noqa: E402
from oracle import Reference  # noqa: E402


def main(n_warps=32768):
    darm.init()
    ref = Reference()
    threads = os.cpu_count() or 1
    for name, meld in (("sb1", 0), ("sb1", 1), ("sb3", 0), ("bitonic", 0), ("nested", 1)):
        mod = ref.load(name, meld)
        prog = darm.Program(mod.text())
        args = np.zeros((len(mod.params), n_warps), np.int32)
        gl = np.zeros((n_warps, prog.global_words), np.int32)
        sh = np.zeros((n_warps, max(1, prog.shared_words)), np.int32)
        for w in range(n_warps):
            a, g, s = mod.make_random_input(32, 1000 + w)
            args[:, w] = a
            gl[w] = g[: prog.global_words]
            sh[w, : prog.shared_words] = s[: prog.shared_words]
        shv = sh[:, : prog.shared_words].copy() if prog.shared_words else None
        g_ref = gl.copy()
        t0 = time.perf_counter()
        mod.execute_program(32, n_warps, args, g_ref, None if shv is None else shv.copy(), threads=threads)
        cpu_s = time.perf_counter() - t0
        g_gpu = torch.from_numpy(gl).cuda()
        s_gpu = None if shv is None else torch.from_numpy(shv).cuda()
        ts = []
        for i in range(4):
            g_gpu.copy_(torch.from_numpy(gl))
            res = prog.execute_warps(32, args, g_gpu, s_gpu, n_warps=n_warps)
            if i:
                ts.append(res.call_stats["kernel_ms"])
        assert (g_gpu.cpu().numpy() == g_ref).all()
        gpu_ms = min(ts)
        print(f"{name}{'.melded' if meld else ''}: {n_warps} warps  reference {cpu_s * 1e3:.1f} ms on {threads} threads"
              f"  GPU {gpu_ms:.3f} ms  ({cpu_s * 1e3 / gpu_ms:.0f}x)  {n_warps / gpu_ms * 1e3:.3e} warps/s", flush=True)


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
