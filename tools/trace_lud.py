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


def super_steps(path="gpurun_out/trace_lud.json"):
    """Per super-step timeline from a trace: the band (trailing-update kernel
    on the panel stream), the four panels, the far block (on the main stream)."""
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    panel_stream = next(e["args"].get("stream") for e in ev if "panel" in e["name"] and e["ts"] > ev[5]["ts"])
    bands = [e for e in ev if "far" in e["name"] and e["args"].get("stream") == panel_stream]
    fars = [e for e in ev if "far" in e["name"] and e["args"].get("stream") != panel_stream]
    panels = [e for e in ev if "panel" in e["name"]][4:]          # super-step 0's panels run first
    print(f"panel stream {panel_stream}: {len(bands)} bands, {len(fars)} far blocks, {len(panels)} panels")
    for g in (0, 10, 30, 50, 70, 90, 110, 120):
        if g >= len(bands):
            continue
        b = bands[g]
        ps = panels[4 * g:4 * g + 4]
        f = fars[g] if g < len(fars) else None
        r = lambda e: f"[{(e['ts'] - t0):9.1f}, {(e['ts'] + e['dur'] - t0):9.1f}]"  # noqa: E731
        print(f"  g={g:3d} band {r(b)} panels {r(ps[0])[:11]}..{r(ps[-1])[11:]} far {r(f) if f else '-'}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "steps":
        super_steps(*sys.argv[2:])
    else:
        main(*[int(x) for x in sys.argv[1:]])
