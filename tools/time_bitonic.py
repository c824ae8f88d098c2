"""Time the bitonic (or, with --oddeven, the PCM odd-even) bucket sort, every
form (unmelded IPDOM, melded, predicated, bitonic: literal App. A.2) and every
keys-per-thread shape, on cuda:0.

    python tools/time_bitonic.py [--oddeven] [bucket ...]      (run under gpurun)
L2 is flushed (256 MiB write) before every timed launch; min and mean of 10.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402


def main(*buckets, sort=None):
    sort = sort or darm.bitonic_sort
    darm.init()
    s = torch.cuda.current_stream()
    n = 1 << 24
    g = torch.Generator(device="cuda").manual_seed(1234)
    pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    work = torch.empty_like(pristine)
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for B in buckets or (64,):
        want = torch.sort(pristine.view(-1, B), dim=1).values.view(-1)
        wide = 256 if sort is darm.bitonic_sort else 32
        for kpt in (1, 4, 8, 16):
            if kpt == 1 and B > 1024:
                continue
            if kpt > 1 and (kpt > B or B // kpt > wide):
                continue
            res = {}
            forms = (0, 1, 2, 3) if sort is darm.bitonic_sort else (0, 1, 2)
            for v in forms:
                call = sort(work, B, v, stream=s.cuda_stream, want_stats=False, prepare_only=True,
                            keys_per_thread=kpt)
                ts = []
                for i in range(13):
                    work.copy_(pristine)
                    flush.fill_(i)
                    torch.cuda._sleep(100_000)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    call()
                    e1.record(s)
                    torch.cuda.synchronize()
                    if i >= 3:
                        ts.append(e0.elapsed_time(e1) * 1e3)
                assert torch.equal(work, want), (B, kpt, v)
                res[v] = (min(ts), sum(ts) / len(ts))
            gbs = 8 * n / (res[1][1] * 1e-6) / 1e9
            names = {0: "unmelded", 1: "melded", 2: "predicated", 3: "literal"}
            cols = "  ".join(f"{names[v]} {res[v][1]:7.1f} us (min {res[v][0]:6.1f})" for v in forms)
            print(f"{sort.__name__} B={B} kpt={kpt:2d} {cols}  melded/unmelded {res[0][1] / res[1][1]:.3f}"
                  f"  melded {gbs:6.0f} GB/s", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    fn = darm.oddeven_sort if "--oddeven" in args else darm.bitonic_sort
    main(*(int(x) for x in args if x != "--oddeven"), sort=fn)
