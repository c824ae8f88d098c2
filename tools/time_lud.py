"""Time LUD (both forms) on cuda:0 through the prepared C-ABI call (run under gpurun)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402


def main(*sizes):
    darm.init()
    s = torch.cuda.current_stream()
    for n in sizes or (2048, 4096, 8192):
        g = torch.Generator(device="cuda").manual_seed(4)
        a0 = torch.rand((n, n), generator=g, device="cuda") + n * torch.eye(n, device="cuda")
        a = torch.empty_like(a0)
        res = {}
        outs = {}
        for v in (darm.UNMELDED, darm.MELDED):
            call = darm.lud(a, v, stream=s.cuda_stream, want_stats=False, prepare_only=True)
            ts = []
            for i in range(6):
                a.copy_(a0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                call()
                e1.record(s)
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            res[v] = min(ts)
            outs[v] = a.clone()
        same = torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))
        tf = (2.0 / 3.0) * n ** 3 / (res[1] * 1e-3) / 1e12
        print(f"n={n} unmelded {res[0]:.3f} ms melded {res[1]:.3f} ms speedup {res[0] / res[1]:.3f} "
              f"melded {tf:.1f} TFLOP/s forms_bit_identical={same}", flush=True)


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
