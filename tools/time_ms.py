"""Time MS (bottom-up merge sort, both forms) on cuda:0 through the prepared C-ABI call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402


def main(*sizes):
    darm.init()
    s = torch.cuda.current_stream()
    for n in sizes or (1 << 20, 1 << 24):
        g = torch.Generator(device="cuda").manual_seed(9)
        pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        work = torch.empty_like(pristine)
        want = torch.sort(pristine).values
        res = {}
        for v in (darm.UNMELDED, darm.MELDED):
            call = darm.merge_sort(work, v, stream=s.cuda_stream, want_stats=False, prepare_only=True)
            ts = []
            for i in range(8):
                work.copy_(pristine)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                call()
                e1.record(s)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            assert torch.equal(work, want), (n, v)
            res[v] = sum(ts) / len(ts)
        print(f"merge_sort n={n} unmelded {res[0]:.1f} us melded {res[1]:.1f} us speedup {res[0] / res[1]:.3f} "
              f"melded {n / res[1]:.1f} Mkeys/s", flush=True)


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
