#!/usr/bin/env python3
"""bench.py — the driver's benchmark contract for the DARM runtime path on B200.

Default workload (BASELINE.json configs[1], the metric's config that fits one
GPU): bitonic sort of 2^24 int32 keys per GPU in 64-key buckets, every bucket
sorted by chaining the corpus compare-exchange step (corpus/bitonic.ir), in the
MELDED form; the UNMELDED form is timed in the same run and the speed-up
reported.  One process per GPU (torchrun); the buckets are independent, so each
rank sorts its own keys with no collective ("scaling": "weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload bitonic|sb1|...]

Timing: W untimed warm-up steps, then K steps, each timed with CUDA events on
the launching stream; before every timed step the input is restored from a
pristine copy and L2 is flushed by writing 256 MiB, both outside the events.
The max over ranks of the summed step time gives `value`.  `e2e` times the
public C-ABI call with pinned HOST buffers (H2D + kernel + D2H, library
events).  `--impl reference` times the reference's own CPU path (oracle/_ref:
executeWarp chained over bitonic.ir steps) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Melded vs unmelded speedup & SIMT lane efficiency per kernel, 1-8 B200"
L2_FLUSH_BYTES = 256 << 20


def sm_max_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except Exception:
        return 1965.0


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


LANE_KEYS = {"nqueens16": "nqueens", "nqueens16_paper_shape": "nqueens_paper_shape", "pcm": "pcm_16kpt", "pcm_1key": "pcm_1kpt", "ms1m": "ms",
             "lud8192": "lud_panel", "srad16384x100": "srad", "srad16384x100_fast_math": "srad_fast",
             "bitonic": "bitonic_sort_16kpt", "bitonic_1key": "bitonic_sort_1kpt"}


def attach_lane_efficiency(per_kernel):
    """SIMT lane efficiency of every per-kernel row from the committed ncu sweep
    (profiles/r<NN>_lane_efficiency.json, tools/lane_eff.sh) and, for the corpus
    kernels, the reference simulator's unit-latency utilisation in the same
    configuration (profiles/r<NN>_simulator_util.json, oracle/sim_util.py)."""
    import glob

    def latest(stem):
        paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r[0-9][0-9]_{stem}.json")))
        if not paths:
            return None, None
        with open(paths[-1]) as f:
            return json.load(f), os.path.relpath(paths[-1], ROOT)

    le, le_src = latest("lane_efficiency")
    sim, sim_src = latest("simulator_util")
    for key, row in per_kernel.items():
        k = LANE_KEYS.get(key, key)
        if le and k in le["kernels"]:
            e = le["kernels"][k]
            row["lane_efficiency"] = {
                form: {"thread_inst_per_inst_div32": round(e[form]["lane_efficiency"], 4),
                       "pred_on_div32": round(e[form]["lane_efficiency_pred_on"], 4)}
                for form in ("unmelded", "predicated", "melded", "melded_literal") if form in e}
            row["lane_efficiency"]["source"] = le_src
        sk = "bitonic_step" if key == "bitonic_step" else key
        if sim and sk in sim["utilization"]:
            row["reference_simulator_utilization"] = dict(sim["utilization"][sk], source=sim_src)


def ncu_kernel_summary(stem, pattern):
    """Latest committed ncu summary profiles/r<NN>_ncu_<stem>.json -> entry whose
    kernel name contains `pattern` (None when absent)."""
    import glob

    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r[0-9][0-9]_ncu_{stem}.json")))
    if not paths:
        return None, None
    with open(paths[-1]) as f:
        d = json.load(f)
    for k in d.get("kernels", []):
        if pattern in k.get("kernel", ""):
            return k, os.path.relpath(paths[-1], ROOT)
    return None, os.path.relpath(paths[-1], ROOT)


def roof(bound, achieved, peak, unit, **extra):
    """A per-kernel roofline object: achieved / peak of the binding roof."""
    d = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
         "frac": (achieved / peak) if (achieved is not None and peak) else None}
    d.update(extra)
    return d


def issue_roof(stem, pattern, seconds, sms, mhz, **extra):
    """Instruction-issue roof: warp instructions of one launch (the committed
    ncu summary of the same launch shape) / the live device time, against
    4 warp instructions per clock per SM (one per scheduler)."""
    prof, src = ncu_kernel_summary(stem, pattern)
    if not prof or not prof.get("warp_inst_executed") or not seconds:
        return roof("issue", None, None, "warp-inst/s", source=src, note="no ncu summary for this kernel")
    peak = 4.0 * sms * mhz * 1e6
    return roof("issue", prof["warp_inst_executed"] / seconds, peak, "warp-inst/s",
                warp_inst_per_launch=prof["warp_inst_executed"], source=src,
                issue_active_pct_ncu=prof.get("issue_active_pct"), **extra)


def cpu_threads():
    return os.cpu_count() or 1


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) is polled every 0.5 ms from a thread, so even a
    few-millisecond timed region yields samples; nvidia-smi (100 ms) is the
    fallback when NVML is unavailable."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []          # (sm_mhz, max_mhz, set of reason names)
        self.stop = threading.Event()
        self.thread = None
        self.proc = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), float(mx), {n for n, b in bits.items() if r & b}))
                    except Exception:
                        pass
                    time.sleep(0.0005)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            pass
        try:
            fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                      "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={fields}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

            def read():
                for line in self.proc.stdout:
                    p = [x.strip() for x in line.split(",")]
                    if len(p) == 6 and p[0].replace(".", "").isdigit():
                        self.samples.append((float(p[0]), float(p[1]),
                                             {n for n, v in zip(self.NAMES, p[2:]) if v.lower() == "active"}))

            self.thread = threading.Thread(target=read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*(s[2] for s in self.samples))),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ timing
def time_steps(torch, stream, prepare, step, steps, warmup, flush_buf):
    """Per-step CUDA-event timing on `stream`; prepare() and the L2 flush run
    before each step outside the events.  Returns the list of step times (ms)."""
    for _ in range(warmup):
        prepare()
        step()
    torch.cuda.synchronize()
    times = []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        prepare()
        flush_buf.fill_(i & 0xFF)  # write 256 MiB > 126 MB L2
        torch.cuda._sleep(200_000)  # keep the GPU busy while the host enqueues step()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    for a, b in evs:
        times.append(a.elapsed_time(b))
    return times


def reduce_max(torch, dist, value):
    if dist is None:
        return value
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ reference arm
def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Reference, Restatement, reference_available

    threads = os.cpu_count() or 1
    B = args.bucket
    n_sample = args.ref_sample_buckets * B
    rng = np.random.default_rng(0)
    keys0 = rng.integers(-(2 ** 31), 2 ** 31, size=n_sample, dtype=np.int64).astype(np.int32)
    if reference_available() and B <= 64:
        kind = "reference"
        mod = Reference().load("bitonic", 0)
        run = lambda k: mod.bitonic_sort(k, B, threads=threads)  # noqa: E731
        what = f"oracle/_ref: reference executeWarp chained over bitonic.ir steps, {threads} threads"
    else:
        kind = "port"
        ora = Restatement()
        run = lambda k: ora.bitonic_sort(k, B)  # noqa: E731
        threads = 1
        what = "oracle restatement (darm_oracle.c), 1 thread"
    for _ in range(args.warmup):
        run(keys0.copy())
    times = []
    for _ in range(args.steps):
        k = keys0.copy()
        t0 = time.perf_counter()
        run(k)
        times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    value = n_sample / sec
    sample = f"{args.ref_sample_buckets} buckets x {B} keys ({n_sample} keys) per step of the {args.keys}-key workload"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": workload_config(args, "unmelded"),
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": threads, "kind": kind, "sample": sample,
                         "what": what},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_config(args, variant):
    return {"workload": f"bitonic sort, {args.keys} int32 keys per GPU in {args.bucket}-key buckets "
                        f"(corpus bitonic.ir compare-exchange step chained over every stage)",
            "keys_per_gpu": args.keys, "bucket": args.bucket, "variant": variant,
            "keys_per_thread": args.keys_per_thread or "auto (16)",
            "form": "melded = the order-flip form (`up` folded into the keys); per_kernel.*.melded_literal_us is "
                    "App. A.2's select chain",
            "global_batch": args.keys * int(os.environ.get("WORLD_SIZE", "1")), "parallelism": f"dp{args.gpus} (independent buckets)",
            "l2": "flushed (256 MiB write) before every timed step; input restored from a pristine copy"}


def cpu_baseline(args):
    """The reference itself (oracle/_ref: executeWarp chained over bitonic.ir
    steps) on all host cores, on a bounded sample of the workload: batches of
    4096 buckets until about args.cpu_seconds of CPU work."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Reference, reference_available

    if not (reference_available() and args.bucket <= 64):
        return None
    threads = os.cpu_count() or 1
    B = args.bucket
    nb = args.ref_sample_buckets
    rng = np.random.default_rng(1)
    mod = Reference().load("bitonic", 0)
    mod.bitonic_sort(rng.integers(-(2 ** 31), 2 ** 31, size=8 * B, dtype=np.int64).astype(np.int32), B,
                     threads=threads)
    done, sec = 0, 0.0
    while sec < args.cpu_seconds:
        keys = rng.integers(-(2 ** 31), 2 ** 31, size=nb * B, dtype=np.int64).astype(np.int32)
        t0 = time.perf_counter()
        mod.bitonic_sort(keys, B, threads=threads)
        sec += time.perf_counter() - t0
        done += nb
        assert (keys.reshape(-1, B)[:, 1:] >= keys.reshape(-1, B)[:, :-1]).all()
    return {"value": done * B / sec, "unit": "keys/s", "cores": threads, "kind": "reference",
            "sample": f"{done} buckets x {B} keys ({done * B} keys) through oracle/_ref executeWarp chains, "
                      f"{sec:.1f} s on {threads} threads"}


# ------------------------------------------------------------------ per-kernel table
CORPUS_LANE = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested"]
NQ_NODES_16 = 1141190303
# nodes below the 7-row prefixes of the mirror-symmetric search (row-0 queen in
# columns 0..7) — the GPU's work per N=16 solve (oracle restatement count)
NQ_MIRROR_NODES = 568094534
# A divergent diamond written for this row (not a corpus file): the GPU
# interpreter runs it from IR text like any reference module.
DIAMOND_IR = """global x[64]
global y[64]
global z[64]
fn diamond(%n) {
^e:
  %t = tid
  %c = icmp.lt %t %n
  condbr %c ^l ^r
^l:
  %a = load.global x %t
  %b = mul %a 5
  %d = load.global y %t
  %s = sub %b %d
  store.global z %t %s
  br ^j
^r:
  %a2 = load.global x %t
  %b2 = shl %a2 2
  %d2 = load.global y %t
  %s2 = add %b2 %d2
  store.global z %t %s2
  br ^j
^j:
  ret
}
"""


# ------------------------------------------------------------------ CPU baselines (rank 0, N=1)
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    return oracle


def cpu_corpus(kernel, nw):
    """Config 1 CPU path: the reference's executeWarp (oracle/_ref, unmodified
    interp.cpp) over all nw makeRandomInput warps of the original and of the
    runDarm-melded module on all host threads, plus its compareRuns per warp
    (darm_cli.cpp:250-263's benchOne loop)."""
    o = _oracle()
    if not o.reference_available():
        return None
    import paper_2107_05681_b200 as darm

    ref = o.Reference()
    b = darm.make_random_input(kernel, 32, nw, 1000)
    names = [n for n, _ in ref.load(kernel, 0).globals]
    g0 = np.concatenate([b.globals[n] for n in names])
    from tools.time_corpus import corpus_args

    args = np.array(corpus_args(kernel), np.int32)                 # [param][set]: the GPU rows' split
    th = cpu_threads()
    res, out = {}, {}
    for form, meld in (("unmelded", 0), ("melded", 1)):
        mod = ref.load(kernel, meld)
        g = g0.copy()
        t0 = time.perf_counter()
        f, _ = mod.execute_warps(32, nw, args, g, 32, None, threads=th, want_stats=False)
        res[form] = time.perf_counter() - t0
        out[form] = (g, f)
    mod = ref.load(kernel, 0)
    w, _ = ref.compare_warps(mod, 32, nw, 32, out["unmelded"][0], out["unmelded"][1], out["melded"][0],
                             out["melded"][1])
    lanes = nw * 32
    return {"value": lanes / res["melded"], "unit": "lanes/s", "cores": th, "kind": "reference",
            "unmelded_lanes_per_s": lanes / res["unmelded"], "compare_runs_equal": w == -1,
            "sample": f"all {nw} warps x 32 lanes (the full config), oracle/_ref executeWarp of the original and "
                      f"the runDarm-melded module, {th} threads"}


def cpu_nqueens(mirror_prefixes):
    """Config 3 CPU path: the restatement's bitmask DFS (oracle/darm_oracle.c)
    below the same mirror-symmetric 7-row prefixes the GPU searches, all host threads."""
    o = _oracle()
    r = o.Restatement()
    th = cpu_threads()
    t0 = time.perf_counter()
    sols, nodes = r.nqueens_count_threads(16, 7, mirror_prefixes, th)
    sec = time.perf_counter() - t0
    assert 2 * sols == 14772512, sols
    return {"value": nodes / sec, "unit": "nodes/s", "cores": th, "kind": "port", "seconds": sec,
            "solutions_per_s": 2 * sols / sec,
            "sample": f"the full N=16 count by mirror symmetry ({len(mirror_prefixes)} prefixes, {nodes} nodes), "
                      f"{th} threads"}


def _timed_sample(run, seconds):
    """Repeat run() (one bounded batch -> units done) until about `seconds` of
    CPU work; returns (units, seconds)."""
    done, sec = 0, 0.0
    while sec < seconds:
        t0 = time.perf_counter()
        done += run()
        sec += time.perf_counter() - t0
    return done, sec


def cpu_bucket_sort(net, bucket, seconds=2.0):
    """The CPU path of a bucket-sort row.  Buckets of <= 64 keys: the reference
    itself (oracle/_ref executeWarp chained over the IR step: bitonic.ir, or
    this repo's ir/oddeven_step.ir for PCM) on all host threads.  Larger
    buckets exceed the interpreter's 64-lane warp, so the restatement's
    network (oracle/darm_oracle.c, one thread) is timed instead."""
    o = _oracle()
    rng = np.random.default_rng(11)
    th = cpu_threads()
    if bucket <= 64 and o.reference_available():
        ref = o.Reference()
        if net == "bitonic":
            mod = ref.load("bitonic", 0)
            sort = lambda k: mod.bitonic_sort(k, bucket, threads=th)  # noqa: E731
        else:
            with open(os.path.join(ROOT, "paper_2107_05681_b200", "ir", "oddeven_step.ir")) as f:
                mod = ref.load_text(f.read(), 0)
            sched = o.oddeven_schedule(bucket)
            sort = lambda k: mod.chain_sort(k, bucket, sched, threads=th)  # noqa: E731
        kind, cores, nb = "reference", th, 1024
        what = f"oracle/_ref executeWarp chained over {'bitonic.ir' if net == 'bitonic' else 'ir/oddeven_step.ir'}"
    else:
        r = o.Restatement()
        sort = (lambda k: r.bitonic_sort(k, bucket)) if net == "bitonic" else (lambda k: r.oddeven_sort(k, bucket))
        kind, cores, nb = "port", 1, max(64, (1 << 20) // bucket)
        what = "the C restatement's network (oracle/darm_oracle.c), one thread"

    def batch():
        keys = rng.integers(-(2 ** 31), 2 ** 31, size=nb * bucket, dtype=np.int64).astype(np.int32)
        sort(keys)
        assert (keys.reshape(-1, bucket)[:, 1:] >= keys.reshape(-1, bucket)[:, :-1]).all()
        return nb * bucket

    keys_done, sec = _timed_sample(batch, seconds)
    return {"value": keys_done / sec, "unit": "keys/s", "cores": cores, "kind": kind,
            "sample": f"{keys_done // bucket} buckets x {bucket} keys, {what}, {sec:.1f} s"}


def cpu_merge_sort(n=1 << 20, seconds=2.0):
    """MS CPU path: the restatement's bottom-up merge sort (oracle/darm_oracle.c,
    the same passes as ir/merge_step.ir) of 2^20 keys, one thread."""
    r = _oracle().Restatement()
    rng = np.random.default_rng(12)

    def batch():
        keys = rng.integers(-(2 ** 31), 2 ** 31, size=n, dtype=np.int64).astype(np.int32)
        r.merge_sort(keys)
        return n

    keys_done, sec = _timed_sample(batch, seconds)
    return {"value": keys_done / sec, "unit": "keys/s", "cores": 1, "kind": "port",
            "sample": f"{keys_done // n} sorts of {n} keys, the C restatement, {sec:.1f} s"}


def cpu_interp(ir_text, n_warps, seconds=2.0):
    """Interpreter row CPU path: the reference's executeWarp (oracle/_ref) over
    the same 32-lane warps of the IR function, all host threads."""
    o = _oracle()
    if not o.reference_available():
        return None
    mod = o.Reference().load_text(ir_text, 0)
    sizes = {sz for _, sz in mod.globals}
    assert len(sizes) == 1, "equal global sizes (one per-warp stride)"
    gw = sizes.pop()
    rng = np.random.default_rng(13)
    th = cpu_threads()
    args = np.full((1, 1), 16, np.int32)

    def batch():
        g = rng.integers(-128, 129, size=len(mod.globals) * n_warps * gw, dtype=np.int64).astype(np.int32)
        mod.execute_warps(32, n_warps, args, g, gw, None, threads=th, want_stats=False)
        return n_warps

    warps, sec = _timed_sample(batch, seconds)
    return {"value": warps / sec, "unit": "warps/s", "cores": th, "kind": "reference",
            "sample": f"{warps} warps x 32 lanes, oracle/_ref executeWarp, {sec:.1f} s"}


def cpu_lud(n=4096):
    """Config 4 CPU path: the blocked-LU restatement on all host threads, on a
    stated subsample (n^2 instead of 8192^2; flops scale as n^3)."""
    o = _oracle()
    r = o.Restatement()
    th = cpu_threads()
    a = np.random.default_rng(4).random((n, n), dtype=np.float32) + n * np.eye(n, dtype=np.float32)
    t0 = time.perf_counter()
    r.lud(a, threads=th)
    sec = time.perf_counter() - t0
    flop = (2.0 / 3.0) * n ** 3
    return {"value": flop / sec / 1e12, "unit": "TFLOP/s", "cores": th, "kind": "port", "seconds": sec,
            "sample": f"{n}^2 blocked LU ({flop / ((2.0 / 3.0) * 8192 ** 3):.3f} of the 8192^2 flops), {th} threads"}


def cpu_srad(n=16384, iters=3):
    """Config 5 CPU path: the SRAD restatement on all host threads, on the full
    16384^2 image for a stated subsample of the iterations."""
    o = _oracle()
    r = o.Restatement()
    th = cpu_threads()
    j = np.exp(np.random.default_rng(5).random((n, n), dtype=np.float32)).astype(np.float32)
    t0 = time.perf_counter()
    r.srad(j, iters, 0.5, (0, 127, 0, 127), threads=th)
    sec = time.perf_counter() - t0
    return {"value": n * n * iters / sec, "unit": "pixel-iterations/s", "cores": th, "kind": "port",
            "seconds": sec, "sample": f"{n}^2 image, {iters} of the 100 iterations, {th} threads"}


PER_KERNEL_SECTIONS = ("corpus", "nqueens16", "pcm", "ms1m", "interp", "lud8192", "srad", "bitonic")


def per_kernel_table(torch, darm, stream, flush, steps, warmup, peak, dist=None, rank=0, world=1,
                     sections=PER_KERNEL_SECTIONS, srad_n=16384, srad_iters=100, with_cpu=True):
    """Melded vs unmelded device time for every corpus kernel (config 1 shape:
    2^20 lanes = 32,768 warps of makeRandomInput fixtures, half-warp split),
    N-Queens N=16 (config 3), PCM, MS, LUD 8192^2 (config 4) and SRAD
    16384^2 x 100 (config 5).  Every rank runs it: NQU (prefix i on rank
    i % world) and SRAD (row tiles with halo exchange) are sharded over the
    ranks (strong scaling); the other kernels run as replicas.  Times are the
    max over ranks."""
    out = {}

    def tmax(row):
        for key in [k for k in row if k.endswith("_us")]:
            row[key] = reduce_max(torch, dist, row[key])
        return row

    nw = 1 << 15
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = sm_max_mhz()
    cpu = rank == 0 and world == 1 and with_cpu
    if "corpus" in sections:
        # graph replay of 100 launches, each on its own 2^20-lane batch (inputs from HBM)
        from tools.time_corpus import time_corpus

        times = time_corpus(CORPUS_LANE, launches=100, reps=max(3, steps // 4), n_warps=nw)
        for k in CORPUS_LANE:
            info = darm.kernel_info(k)
            row = {f + "_us": times[k][f] for f in ("unmelded", "predicated", "melded")}
            tmax(row)
            row["speedup"] = row["unmelded_us"] / row["melded_us"]
            row["speedup_vs_predicated"] = row["predicated_us"] / row["melded_us"]
            row["timing"] = "CUDA graph of 100 launches on 100 distinct 2^20-lane batches, per-launch mean, best of reps"
            alg = info["lane_bytes"] * nw * 32
            row["roofline"] = roof("hbm", alg / (row["melded_us"] * 1e-6) / 1e9, peak, "GB/s",
                                   algorithmic_bytes_per_launch=alg,
                                   bytes_per_lane=info["lane_bytes"], form="melded")
            if cpu:
                row["cpu_baseline"] = cpu_corpus(k, nw)
            out[k] = row
    # N-Queens N=16: the 7-row prefixes dealt round-robin over the ranks
    row = {}
    for vname, v in ((("unmelded", 0), ("melded", 1)) if "nqueens16" in sections else ()):
        ts = []
        for i in range(warmup + max(3, steps // 4)):
            if dist:
                dist.barrier()
            sols, _, st = darm.nqueens(16, 7, v, rank=rank, world=world, stream=stream.cuda_stream, mirror=True)
            if dist:
                t = torch.tensor([sols], dtype=torch.int64, device="cuda")
                dist.all_reduce(t)
                sols = int(t.item())
            assert sols == 14772512, sols
            if i >= warmup:
                ts.append(st["kernel_ms"])
        row[vname + "_us"] = 1e3 * sum(ts) / len(ts)
        row[vname + "_solutions"] = sols
    if "nqueens16" in sections:
        nqueens_row(torch, dist, row, world, tmax)
        nodes = NQ_MIRROR_NODES
        row["nodes_searched"] = nodes
        row["melded_nodes_per_s"] = nodes / (row["melded_us"] * 1e-6)
        row["roofline"] = issue_roof("nqueens", "nqueens_kernel<1", row["melded_us"] * 1e-6 * world, sms, mhz,
                                     note="integer-issue bound; nodes below the mirror-symmetric 7-row prefixes")
        if cpu:
            o = _oracle()
            pre = o.Restatement().nqueens_prefixes(16, 7, mirror=True)
            row["cpu_baseline"] = cpu_nqueens(pre)
        out["nqueens16"] = row
        # the same search in the paper's shape (ir/nqueens_step.ir: pop / leaf /
        # push, melded by region replication), beside the symmetric encoding
        row = {}
        for vname, v in (("unmelded", 0), ("melded", 1)):
            ts = []
            for i in range(warmup + max(3, steps // 4)):
                if dist:
                    dist.barrier()
                sols, _, st = darm.nqueens(16, 7, v, rank=rank, world=world, stream=stream.cuda_stream, mirror=True,
                                           paper_shape=True)
                if dist:
                    t = torch.tensor([sols], dtype=torch.int64, device="cuda")
                    dist.all_reduce(t)
                    sols = int(t.item())
                assert sols == 14772512, sols
                if i >= warmup:
                    ts.append(st["kernel_ms"])
            row[vname + "_us"] = 1e3 * sum(ts) / len(ts)
        tmax(row)
        row["speedup"] = row["unmelded_us"] / row["melded_us"]
        row["ir"] = "paper_2107_05681_b200/ir/nqueens_step.ir (runDarm: two block-region melds, region replication)"
        row["nodes_searched"] = NQ_MIRROR_NODES
        row["melded_nodes_per_s"] = NQ_MIRROR_NODES / (row["melded_us"] * 1e-6)
        row["roofline"] = issue_roof("nqueens_step", "nqueens_step_kernel<1", row["melded_us"] * 1e-6 * world, sms,
                                     mhz, note="integer-issue bound; the paper-shaped encoding")
        if cpu:
            row["cpu_baseline"] = out["nqueens16"]["cpu_baseline"]
        out["nqueens16_paper_shape"] = row
    if "pcm" in sections or "ms1m" in sections or "interp" in sections:
        pcm_ms_interp_rows(torch, darm, stream, flush, steps, warmup, peak, dist, out, sections, cpu=cpu)
    if "lud8192" in sections:
        lud_row(torch, darm, stream, flush, steps, warmup, dist, out, tmax, cpu)
    if "srad" in sections:
        srad_rows(torch, darm, stream, flush, peak, dist, world, out, tmax, srad_n, srad_iters, cpu)
    return out


def nqueens_row(torch, dist, row, world, tmax):
    tmax(row)
    row["speedup"] = row["unmelded_us"] / row["melded_us"]
    row["melded_solutions_per_s"] = 14772512 / (row["melded_us"] * 1e-6)
    row["prefix_rows"], row["mirror_symmetry"] = 7, True
    row["n_gpus"], row["scaling"] = world, "strong (prefixes sharded over the ranks)"
    row["full_tree_nodes"] = NQ_NODES_16


def pcm_ms_interp_rows(torch, darm, stream, flush, steps, warmup, peak, dist, out, sections, cpu=False):
    def tmax(row):
        for key in [k for k in row if k.endswith("_us")]:
            row[key] = reduce_max(torch, dist, row[key])
        return row

    # PCM (Batcher odd-even merge sort of 64-key buckets, 2^24 keys) and MS (bottom-up
    # merge sort of 2^20 keys, the paper's input size)
    n = 1 << 24
    g = torch.Generator(device="cuda").manual_seed(6)
    pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
    work = torch.empty_like(pristine)
    want = torch.sort(pristine.view(-1, 64), dim=1).values.view(-1)
    for name, kpt in ((("pcm", 0), ("pcm_1key", 1)) if "pcm" in sections else ()):
        row = {}
        for vname, v in (("unmelded", 0), ("predicated", 2), ("melded", 1)):
            call = darm.oddeven_sort(work, 64, v, stream=stream.cuda_stream, want_stats=False, prepare_only=True,
                                     keys_per_thread=kpt)
            t = time_steps(torch, stream, lambda: work.copy_(pristine), call, steps, warmup, flush)
            if not torch.equal(work, want):
                raise SystemExit(f"{name} {vname}: result is not the bucket-sorted input")
            row[vname + "_us"] = 1e3 * sum(t) / len(t)
        tmax(row)
        row["speedup"] = row["unmelded_us"] / row["melded_us"]
        row["speedup_vs_predicated"] = row["predicated_us"] / row["melded_us"]
        row["keys_per_thread"] = kpt or 16
        row["melded_GBps"] = 8.0 * n / (row["melded_us"] * 1e-6) / 1e9
        row["melded_frac_hbm"] = row["melded_GBps"] / peak
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        pat = "oddeven_sort_reg_kernel<1, 64, 16" if kpt == 0 else "oddeven_sort_kernel<1, 64,"
        row["roofline"] = roof("hbm", row["melded_GBps"], peak, "GB/s", algorithmic_bytes_per_launch=8 * n,
                               issue=issue_roof("oddeven", pat, row["melded_us"] * 1e-6, sms, sm_max_mhz()))
        if cpu:
            row["cpu_baseline"] = out["pcm"]["cpu_baseline"] if name == "pcm_1key" else cpu_bucket_sort("oddeven", 64)
        out[name] = row
    n = 1 << 20
    keys = pristine[:n].clone()
    ms = torch.empty_like(keys)
    want = torch.sort(keys).values
    if "ms1m" not in sections:
        return interp_row(torch, darm, dist, steps, warmup, g, out, cpu=cpu) if "interp" in sections else None
    row = {}
    for vname, v in (("unmelded", 0), ("melded", 1)):
        call = darm.merge_sort(ms, v, stream=stream.cuda_stream, want_stats=False, prepare_only=True)
        t = time_steps(torch, stream, lambda: ms.copy_(keys), call, steps, warmup, flush)
        if not torch.equal(ms, want):
            raise SystemExit(f"ms {vname}: result is not sorted")
        row[vname + "_us"] = 1e3 * sum(t) / len(t)
    tmax(row)
    row["speedup"] = row["unmelded_us"] / row["melded_us"]
    row["melded_keys_per_s"] = n / (row["melded_us"] * 1e-6)
    passes = 1 + max(0, (n // 4096).bit_length() - 1)        # tile pass + one per width >= 4096
    row["melded_GBps"] = 8.0 * n * passes / (row["melded_us"] * 1e-6) / 1e9
    row["melded_frac_hbm"] = row["melded_GBps"] / peak
    row["roofline"] = roof("hbm", row["melded_GBps"], peak, "GB/s", algorithmic_bytes_per_launch=8 * n * passes,
                           note=f"8 B/key per pass x {passes} passes; at 2^20 keys (4 MiB) the passes run from L2")
    if cpu:
        row["cpu_baseline"] = cpu_merge_sort(n)
    out["ms1m"] = row
    if "interp" in sections:
        interp_row(torch, darm, dist, steps, warmup, g, out, cpu=cpu)


def interp_row(torch, darm, dist, steps, warmup, g, out, cpu=False):
    # the GPU executeWarp for arbitrary IR (darm_gpu_program_execute): a diamond
    # kernel given as IR text, 32768 warps of 32 lanes (config 1 shape)
    row = {}
    for vname in ("diamond",):
        prog = darm.Program(DIAMOND_IR)
        nwi = 1 << 15
        gi = torch.randint(-128, 129, (nwi, prog.global_words), dtype=torch.int32, device="cuda", generator=g)
        work_g = torch.empty_like(gi)
        argv = np.full((1, 1), 16, np.int32)
        ts = []
        for i in range(warmup + steps):
            work_g.copy_(gi)
            res = prog.execute_warps(32, argv, work_g, n_warps=nwi)
            if i >= warmup:
                ts.append(res.call_stats["kernel_ms"])
        row[vname + "_us"] = reduce_max(torch, dist, 1e3 * sum(ts) / len(ts))
        row[vname + "_warps_per_s"] = nwi / (row[vname + "_us"] * 1e-6)
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    row["roofline"] = issue_roof("interp", "ir_interp_kernel", row["diamond_us"] * 1e-6, sms, sm_max_mhz(),
                                 note="an interpreter: bound by issue per IR instruction, not by bytes")
    if cpu:
        row["cpu_baseline"] = cpu_interp(DIAMOND_IR, 1 << 15)
    out["interp_diamond_32k_warps"] = row


def lud_row(torch, darm, stream, flush, steps, warmup, dist, out, tmax, cpu=False):
    # LUD 8192^2 fp32 (config 4): the whole decomposition (n/16 + 2n/64 + 1 launches in one graph)
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(4)
    a0 = torch.rand((n, n), generator=g, device="cuda") + n * torch.eye(n, device="cuda")
    a = torch.empty_like(a0)
    row = {}
    for vname, v in (("unmelded", 0), ("melded", 1)):
        call = darm.lud(a, v, stream=stream.cuda_stream, want_stats=False, prepare_only=True)
        t = time_steps(torch, stream, lambda: a.copy_(a0), call, max(2, steps // 4), min(warmup, 3), flush)
        row[vname + "_us"] = 1e3 * sum(t) / len(t)
    tmax(row)
    row["speedup"] = row["unmelded_us"] / row["melded_us"]
    row["melded_TFLOPs"] = (2.0 / 3.0) * n ** 3 / (row["melded_us"] * 1e-6) / 1e12
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    roof = sms * 256 * sm_max_mhz() * 1e6 / 1e12             # fp32 FMA: 128 lanes x 2 flop per SM per clock
    row["fp32_roof_TFLOPs"] = roof
    row["melded_frac_fp32"] = row["melded_TFLOPs"] / roof
    row["roofline"] = {"bound": "fp32 FMA (CUDA cores)", "achieved": row["melded_TFLOPs"], "peak": roof,
                       "unit": "TFLOP/s", "frac": row["melded_frac_fp32"],
                       "algorithmic_flop": (2.0 / 3.0) * n ** 3, "peak_source": "SMs x 128 FMA x 2 x sm_max_mhz"}
    pattern = ffma2_outer_product_roof()
    if pattern:
        # the trailing update's instruction pattern (8 x 8 register outer product of
        # FFMA2 with both operands in registers) measured alone on this GPU, no memory
        row["roofline"]["pattern_roof"] = pattern
        row["roofline"]["frac_of_pattern_roof"] = row["melded_TFLOPs"] / pattern["TFLOPs"]
    if cpu:
        row["cpu_baseline"] = cpu_lud()
    out["lud8192"] = row


def ffma2_outer_product_roof():
    """FFMA2 throughput of the LUD far update's register outer product (8 rows
    x 4 column pairs per thread, L broadcast, U and the accumulators in
    registers, no memory traffic) measured now by tools/micro/ffma2_outer; None
    when the binary was not built."""
    exe = os.path.join(ROOT, "tools", "micro", "ffma2_outer")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=60, check=True).stdout
    except (subprocess.SubprocessError, OSError):
        return None
    vals = [float(line.rsplit(":", 1)[1].split()[0]) for line in out.splitlines() if "TFLOP/s" in line]
    if not vals:
        return None
    return {"TFLOPs": max(vals), "source": "tools/micro/ffma2_outer (best of 8 / 16 warps per SM, both operand orders)",
            "note": "an FFMA2 with two register-pair sources issues at about two thirds of the pipe's rate; "
                    "with a uniform-register operand the same pipe reaches ~69 TFLOP/s (tools/micro/ffma2_peak)"}


def srad_rows(torch, darm, stream, flush, peak, dist, world, out, tmax, n=16384, iters=100, cpu=False):
    # SRAD 16384^2 fp32 x 100 iterations (config 5): one GPU, or row tiles with a
    # halo exchange and the ROI all-reduce every iteration over NCCL
    g = torch.Generator(device="cuda").manual_seed(4)
    j0 = torch.exp(torch.rand((n, n), generator=g, device="cuda"))
    import hashlib

    sha = lambda t: hashlib.sha256(t.contiguous().cpu().numpy().tobytes()).hexdigest()[:16]  # noqa: E731
    tag = f"srad{n}x{iters}"
    for key, fast in ((tag, False), (tag + "_fast_math", True)):
        row = {"rows": n, "cols": n, "iters": iters}
        flag = darm.FAST_MATH if fast else 0
        if world == 1:
            j = torch.empty_like(j0)
            for vname, v in (("unmelded", 0), ("melded", 1)):
                call = darm.srad(j, iters, 0.5, darm.RODINIA_ROI, v, stream=stream.cuda_stream, want_stats=False,
                                 prepare_only=True, fast=fast)
                t = time_steps(torch, stream, lambda: j.copy_(j0), call, 2, 1, flush)
                row[vname + "_us"] = 1e3 * sum(t) / len(t)
                row[vname + "_result_sha16"] = sha(j)
            del j
        else:
            from paper_2107_05681_b200.srad_peer import SradPeerTiles
            from paper_2107_05681_b200.srad_tiles import SradTiles

            # the product path: peer-memory tiles, the whole run one CUDA graph per rank
            for vname, v in (("unmelded", 0), ("melded", 1)):
                tiles = SradPeerTiles(n, n, 0.5, darm.RODINIA_ROI, dist=dist, variant=v, fast=fast)
                ts = []
                for rep in range(2):
                    tiles.load(j0)
                    torch.cuda.synchronize()
                    dist.barrier()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    tiles.run(iters)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    if rep:
                        ts.append(e0.elapsed_time(e1))
                row[vname + "_us"] = 1e3 * sum(ts) / len(ts)
                full = tiles.gather()
                if full is not None:
                    row[vname + "_result_sha16"] = sha(full)
                dist.barrier()
                tiles.close()
                del tiles, full
            row["transport"] = "peer memory (CUDA IPC over NVLink), device-flag phases, one CUDA graph"
            # the baseline transport: torch.distributed P2P halos + ROI all-reduce per iteration (melded)
            tiles = SradTiles(n, n, 0.5, darm.RODINIA_ROI, dist=dist, device=torch.device("cuda"),
                              variant=1 | flag)
            tiles.load(j0)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tiles.run(iters)
            e1.record(stream)
            torch.cuda.synchronize()
            row["melded_torch_dist_transport_us"] = reduce_max(torch, dist, 1e3 * e0.elapsed_time(e1))
            full = tiles.gather()
            if full is not None:
                row["melded_torch_dist_result_sha16"] = sha(full)
            del tiles, full
        tmax(row)
        row["speedup"] = row["unmelded_us"] / row["melded_us"]
        # minimal traffic 8 B/px/iteration (one read of J, one write of J') + the in/out copies of the call
        alg = 8.0 * n * n * iters + 8.0 * n * n
        row["melded_GBps"] = alg / (row["melded_us"] * 1e-6) / 1e9
        row["melded_frac_hbm"] = row["melded_GBps"] / (peak * world)
        row["n_gpus"], row["scaling"] = world, ("strong (row tiles, peer-memory halos)" if world > 1 else
                                                "single GPU")
        row["arithmetic"] = ("one reciprocal per pixel, f32x2 FMA (DARM_FAST_MATH), within 1e-5 relative" if fast
                             else "IEEE, bit-exact vs the restatement")
        row["roofline"] = roof("hbm", row["melded_GBps"], peak * world, "GB/s", algorithmic_bytes=alg,
                               bytes_per_px_iter=8, note="one read of J and one write of J' per pixel and iteration")
        row["melded_pixel_iters_per_s"] = n * n * iters / (row["melded_us"] * 1e-6)
        if cpu and fast:
            row["cpu_baseline"] = out[tag]["cpu_baseline"]
        elif cpu:
            row["cpu_baseline"] = cpu_srad()
        out[key] = row
    return out


# ------------------------------------------------------------------ our arm
def our_arm(args):
    import torch

    import paper_2107_05681_b200 as darm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        # DARM_DIST_BACKEND=gloo: a functional run of the multi-rank logic with
        # several ranks on one GPU (NCCL refuses two ranks per device)
        backend = os.environ.get("DARM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist_mod.init_process_group(backend)
        dist = dist_mod
    darm.init()
    stream = torch.cuda.current_stream()
    n, B = args.keys, args.bucket
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    pristine = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=gen)
    work = torch.empty_like(pristine)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    want = torch.sort(pristine.view(-1, B), dim=1).values.view(-1)

    results = {}
    for vname, variant in (("unmelded", darm.UNMELDED), ("melded", darm.MELDED)):
        prepare = lambda: work.copy_(pristine)  # noqa: E731
        step = darm.bitonic_sort(work, B, variant, stream=stream.cuda_stream, want_stats=False, prepare_only=True,
                                 keys_per_thread=args.keys_per_thread)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(dev_index) as clk:
            times = time_steps(torch, stream, prepare, step, args.steps, args.warmup, flush)
        torch.cuda.synchronize()
        if not torch.equal(work, want):
            raise SystemExit(f"bitonic {vname}: result is not the bucket-sorted input")
        total_ms = reduce_max(torch, dist, sum(times))
        results[vname] = {"total_ms": total_ms, "ms_per_step": total_ms / args.steps,
                          "kernel_ms_mean": sum(times) / len(times), "clocks": clk.summary()}
    if dist:
        dist.barrier()

    # e2e: public C-ABI call with pinned host buffers, copies inside the timed region
    host_pristine = pristine.cpu().numpy()
    host = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
    # host wall clock around the (synchronous) call: argument checks, staging,
    # launches and both copies; the library's own events beside it
    e2e_ms, e2e_lib_ms = [], []
    for i in range(args.warmup + args.steps):
        host[:] = host_pristine
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = darm.bitonic_sort(host, B, darm.MELDED, stream=stream.cuda_stream, keys_per_thread=args.keys_per_thread)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_ms.append(1e3 * (t1 - t0))
            e2e_lib_ms.append(st["total_ms"])
    if not (host.reshape(-1, B) == want.view(-1, B).cpu().numpy()).all():
        raise SystemExit("bitonic e2e: result is not the bucket-sorted input")
    e2e_total = reduce_max(torch, dist, sum(e2e_ms))
    e2e_lib_total = reduce_max(torch, dist, sum(e2e_lib_ms))

    kpt = args.keys_per_thread or 16
    per_kernel = None
    if not args.no_per_kernel:
        peak0, _ = measured_peaks()
        sections = tuple(x for x in args.kernels.split(",") if x)
        bad = set(sections) - set(PER_KERNEL_SECTIONS)
        if bad:
            raise SystemExit(f"unknown --kernels {sorted(bad)}; choose from {PER_KERNEL_SECTIONS}")
        try:
            per_kernel = per_kernel_table(torch, darm, stream, flush, args.steps, args.warmup, peak0, dist, rank,
                                          world, sections, args.srad_size, args.srad_iters,
                                          with_cpu=not args.no_cpu_baseline)
        except Exception as e:          # the per-kernel table is auxiliary: the headline line still prints
            if world == 1:
                raise
            per_kernel = {"error": f"{type(e).__name__}: {e}"[:400]}
            sections = ()
    if per_kernel is not None and "error" not in per_kernel and "bitonic" in sections:
        # every shape in four forms: unmelded (IPDOM branches), predicated
        # (ptxas if-conversion of the same CFG), melded (the order-flip form the
        # headline reports: `up` folded into the data) and melded_literal (App.
        # A.2's select chain on `up` as runDarm prints it) — the literal form
        # isolates the melding gain, the order-flip form adds the data rewrite
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        forms = (("unmelded", darm.UNMELDED), ("predicated", darm.PREDICATED), ("melded", darm.MELDED),
                 ("melded_literal", darm.MELDED_LITERAL))
        shapes = [("bitonic", B, 0), ("bitonic_1key", B, 1)] + [(f"bitonic_B{b}", b, 0) for b in (256, 1024, 4096)] + \
                 [(f"bitonic_B{b}_1key", b, 1) for b in (256, 1024)]
        cpu_rows = {}
        for key, Bs, kp in shapes:
            want_s = want if Bs == B else torch.sort(pristine.view(-1, Bs), dim=1).values.view(-1)
            row = {}
            for vname, variant in forms:
                if key == "bitonic" and vname in ("unmelded", "melded") and kp == (args.keys_per_thread or 0):
                    row[vname + "_us"] = 1e3 * results[vname]["kernel_ms_mean"]
                    continue
                step = darm.bitonic_sort(work, Bs, variant, stream=stream.cuda_stream, want_stats=False,
                                         prepare_only=True, keys_per_thread=kp)
                t = time_steps(torch, stream, lambda: work.copy_(pristine), step, args.steps, args.warmup, flush)
                if not torch.equal(work, want_s):
                    raise SystemExit(f"{key} {vname}: result is not the bucket-sorted input")
                row[vname + "_us"] = reduce_max(torch, dist, 1e3 * sum(t) / len(t))
            row["speedup"] = row["unmelded_us"] / row["melded_us"]
            row["speedup_literal"] = row["unmelded_us"] / row["melded_literal_us"]
            row["speedup_vs_predicated"] = row["predicated_us"] / row["melded_us"]
            row["keys_per_thread"] = kp or 16
            row["bucket"] = Bs
            gbs = 8 * n / (row["melded_us"] * 1e-6) / 1e9
            kpt_name = f"bitonic_sort_reg_kernel<1, {Bs}, 16" if kp != 1 else f"bitonic_sort_kernel<1, {Bs},"
            stem = "bitonic" if Bs == 64 else f"bitonic_b{Bs}"
            row["roofline"] = roof("hbm", gbs, peak0, "GB/s", algorithmic_bytes_per_launch=8 * n, form="melded",
                                   issue=issue_roof(stem, kpt_name, row["melded_us"] * 1e-6, sms, sm_max_mhz()))
            if world == 1 and not args.no_cpu_baseline:
                # the CPU path does not depend on the GPU shape: one sample per bucket size
                cpu_rows.setdefault(Bs, cpu_bucket_sort("bitonic", Bs))
                row["cpu_baseline"] = cpu_rows[Bs]
            per_kernel[key] = row

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    mel, unm = results["melded"], results["unmelded"]
    value = n * world / (mel["total_ms"] / args.steps / 1e3)
    peak, peak_src = measured_peaks()
    alg_bytes = 8 * n
    achieved = alg_bytes / (mel["kernel_ms_mean"] / 1e3) / 1e9
    kname = "bitonic_sort_reg_kernel<{}, %d, %d" % (B, kpt) if kpt > 1 else "bitonic_sort_kernel<{}, %d" % B
    prof_m, prof_src = ncu_kernel_summary("bitonic", kname.format(1))
    prof_u, _ = ncu_kernel_summary("bitonic", kname.format(0))
    lane_eff = None
    if prof_m and prof_u:
        lane_eff = {"source": prof_src + " (ncu --set full, one launch per form)",
                    "unmelded": {"thread_inst_per_inst_div32": prof_u.get("lane_efficiency"),
                                 "pred_on_div32": prof_u.get("lane_efficiency_pred_on"),
                                 "branch_uniform_pct": prof_u.get("branch_uniform_pct")},
                    "melded": {"thread_inst_per_inst_div32": prof_m.get("lane_efficiency"),
                               "pred_on_div32": prof_m.get("lane_efficiency_pred_on"),
                               "branch_uniform_pct": prof_m.get("branch_uniform_pct")}}
    line = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mel["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic (uniform full-range int32, torch.randint)",
        "config": workload_config(args, "melded"),
        "melded_vs_unmelded_speedup": unm["total_ms"] / mel["total_ms"],
        "unmelded": {"value": n * world / (unm["total_ms"] / args.steps / 1e3), "ms_per_step": unm["ms_per_step"]},
        "lane_efficiency": lane_eff,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (prof_m or {}).get("dram_bytes"), "peak_source": peak_src,
                     "traffic_note": "ncu dram__bytes read+write of one launch; below the algorithmic bytes "
                                     "because the written keys stay in the 126 MB L2 at kernel end",
                     "kernel": kname.format("true"),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "alu_pipe_pct": (prof_m or {}).get("alu_pipe_pct"),
                     "issue": issue_roof("bitonic", kname.format(1), mel["kernel_ms_mean"] / 1e3,
                                         torch.cuda.get_device_properties(torch.cuda.current_device())
                                         .multi_processor_count, sm_max_mhz()),
                     "note": "instruction-issue-bound (VIMNMX compare-exchanges on the ALU pipe, half the "
                             "in-register maxima as IMADs on the FMA pipe, 21 steps per key): the `issue` object is "
                             "the binding roof; see DESIGN.md §5"},
        "e2e": {"value": n * world / (e2e_total / args.steps / 1e3), "unit": "keys/s",
                "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
                "how": "darm_gpu_bitonic_sort(mem=HOST) on pinned numpy buffers; host wall clock around the "
                       "synchronous call (H2D, sort and D2H pipelined in 2^21-key chunks inside it)",
                "library_events_keys_per_s": n * world / (e2e_lib_total / args.steps / 1e3)},
        "gpu_launches": args.steps,
        "clocks": mel["clocks"],
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if per_kernel is not None:
        if "error" not in per_kernel:
            attach_lane_efficiency(per_kernel)
        line["per_kernel"] = per_kernel
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1 with this same command
    line; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--keys", type=int, default=1 << 24)
    ap.add_argument("--bucket", type=int, default=64)
    ap.add_argument("--ref-sample-buckets", type=int, default=4096)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--keys-per-thread", type=int, default=0, help="0 = auto (16), 1 = one key per thread")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-kernel", action="store_true")
    ap.add_argument("--kernels", default=",".join(PER_KERNEL_SECTIONS),
                    help="per-kernel table sections (comma list of %s)" % ",".join(PER_KERNEL_SECTIONS))
    ap.add_argument("--srad-size", type=int, default=16384)
    ap.add_argument("--srad-iters", type=int, default=100)
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
