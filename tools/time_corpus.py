"""Corpus kernels at 2^20 lanes (config 1 shape), every form, by CUDA-graph
replay (run under gpurun).

Each form is timed as one graph of `launches` back-to-back launches, each on
its own 2^20-lane batch (distinct buffers: 100 batches of sb1 are 1.6 GB, far
above the 126 MB L2, so every launch reads its inputs from HBM); the figure is
graph time / launches, so launch latency is amortised.

    python tools/time_corpus.py [--launches 100] [--reps 5]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402

CORPUS_LANE = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested"]
FORMS = (("unmelded", darm.UNMELDED), ("predicated", darm.PREDICATED), ("melded", darm.MELDED))


def corpus_args(kernel):
    """The half-warp split of acceptance.cpp:251-253 (sb4: h = 16, q = 24)."""
    return [[16], [24]] if kernel in ("sb4", "sb4r") else [[16]]


def graph_time_us(kernel, variant, batches, args, launches, reps, flush):
    """Mean device time per launch (µs) of a graph of `launches` launches,
    best of `reps` replays, L2 flushed before each replay."""
    stream = torch.cuda.Stream()
    calls = [darm.execute_warps(kernel, variant, 32, args, g, want_stats=False, stream=stream.cuda_stream,
                                prepare_only=True, count_faults=False) for g in batches]
    with torch.cuda.stream(stream):
        for c in calls[:3]:
            c()                                   # warm-up outside the capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for i in range(launches):
            calls[i % len(calls)]()
    best = float("inf")
    for _ in range(reps):
        flush.fill_(7)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / launches)
    return best


def time_corpus(kernels=CORPUS_LANE, launches=100, reps=5, n_warps=1 << 15, split=None):
    """{kernel: {form: µs per launch}} for the 2^20-lane corpus batches."""
    darm.init()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    out = {}
    for k in kernels:
        b = darm.make_random_input(k, 32, n_warps, 1000)
        nb = min(launches, 100)
        batches = [{n: torch.from_numpy(a).cuda() for n, a in b.globals.items()} for _ in range(nb)]
        args = corpus_args(k) if split is None else [[split]]
        out[k] = {name: graph_time_us(k, v, batches, args, launches, reps, flush) for name, v in FORMS}
        del batches
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=100)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    res = time_corpus(launches=a.launches, reps=a.reps)
    for k, r in res.items():
        print(f"{k:8s} unmelded {r['unmelded']:6.2f} us  predicated {r['predicated']:6.2f} us  "
              f"melded {r['melded']:6.2f} us  speedup vs unmelded {r['unmelded'] / r['melded']:.3f}  "
              f"vs predicated {r['predicated'] / r['melded']:.3f}", flush=True)
    # sb1 with the split point n swept over the warp
    # (n = 0 and 32: no divergence; 16: half the warp each way)
    for split in (0, 8, 16, 24, 32):
        r = time_corpus(["sb1"], a.launches, a.reps, split=split)["sb1"]
        print(f"sb1 n={split:2d} unmelded {r['unmelded']:6.2f} us  predicated {r['predicated']:6.2f} us  "
              f"melded {r['melded']:6.2f} us  speedup {r['unmelded'] / r['melded']:.3f}", flush=True)


if __name__ == "__main__":
    main()
