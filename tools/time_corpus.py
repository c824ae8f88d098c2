"""Corpus kernels at 2^20 lanes (config 1 shape), both forms, as bench.py's
per-kernel rows (run under gpurun)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2107_05681_b200 as darm  # noqa: E402


def main(steps=50, warmup=10):
    darm.init()
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    nw = 1 << 15
    for k in bench.CORPUS_LANE:
        b = darm.make_random_input(k, 32, nw, 1000)
        g = {n: torch.from_numpy(a).cuda() for n, a in b.globals.items()}
        args = [[16]] if len(b.args) == 1 else [[16], [24]]
        row = {}
        for vname, v in (("unmelded", 0), ("melded", 1)):
            step = darm.execute_warps(k, v, 32, args, g, want_stats=False, stream=stream.cuda_stream,
                                      prepare_only=True)
            t = bench.time_steps(torch, stream, lambda: None, step, steps, warmup, flush)
            row[vname] = 1e3 * sum(t) / len(t)
        print(f"{k:8s} unmelded {row['unmelded']:7.2f} us  melded {row['melded']:7.2f} us  "
              f"speedup {row['unmelded'] / row['melded']:.3f}", flush=True)
    # sb1 with the split point n swept over the warp
    # (n = 0 and 32: no divergence; 16: half the warp each way)
    b = darm.make_random_input("sb1", 32, nw, 1000)
    g = {n: torch.from_numpy(a).cuda() for n, a in b.globals.items()}
    for split in (0, 8, 16, 24, 32):
        row = {}
        for vname, v in (("unmelded", 0), ("melded", 1)):
            step = darm.execute_warps("sb1", v, 32, [[split]], g, want_stats=False, stream=stream.cuda_stream,
                                      prepare_only=True)
            t = bench.time_steps(torch, stream, lambda: None, step, steps, warmup, flush)
            row[vname] = 1e3 * sum(t) / len(t)
        print(f"sb1 n={split:2d} unmelded {row['unmelded']:7.2f} us  melded {row['melded']:7.2f} us  "
              f"speedup {row['unmelded'] / row['melded']:.3f}", flush=True)


if __name__ == "__main__":
    main()
