"""Kernel timeline of one LUD call (torch.profiler / CUPTI, run under gpurun):
per-kernel start/end, to see what overlaps inside the recorded graph."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402


def main(n=8192, variant=1, out="gpurun_out/trace_lud.json"):
    darm.init()
    s = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(4)
    a0 = torch.rand((n, n), generator=g, device="cuda") + n * torch.eye(n, device="cuda")
    a = torch.empty_like(a0)
    call = darm.lud(a, variant, stream=s.cuda_stream, want_stats=False, prepare_only=True)
    for _ in range(2):
        a.copy_(a0)
        call()
    torch.cuda.synchronize()
    a.copy_(a0)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        call()
        torch.cuda.synchronize()
    prof.export_chrome_trace(out)
    ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    span = ev[-1]["ts"] + ev[-1]["dur"] - t0
    by = {}
    for e in ev:
        k = "far" if "far" in e["name"] else "panel" if "panel" in e["name"] else e["name"][:30]
        by.setdefault(k, []).append(e)
    print(f"n={n} span {span / 1e3:.3f} ms, {len(ev)} kernels")
    for k, es in by.items():
        print(f"  {k}: {len(es)} launches, sum {sum(e['dur'] for e in es) / 1e3:.3f} ms")
    # busy union and panel time overlapped with a far kernel
    far = sorted((e["ts"], e["ts"] + e["dur"]) for e in by.get("far", []))
    ov = 0.0
    for e in by.get("panel", []):
        a_, b_ = e["ts"], e["ts"] + e["dur"]
        for f0, f1 in far:
            ov += max(0.0, min(b_, f1) - max(a_, f0))
    print(f"  panel time overlapped with far: {ov / 1e3:.3f} ms")
    # first groups in detail
    for e in ev[:24]:
        print(f"    {(e['ts'] - t0):9.1f} +{e['dur']:7.1f} us  stream {e['args'].get('stream')}  {e['name'][:60]}")
    gaps = 0.0
    end = ev[0]["ts"]
    for e in ev:
        if e["ts"] > end:
            gaps += e["ts"] - end
        end = max(end, e["ts"] + e["dur"])
    print(f"  idle gaps (no kernel running): {gaps / 1e3:.3f} ms")


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
