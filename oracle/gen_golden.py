"""Generate tests/golden/*.json by running the UNMODIFIED reference.

TEST INFRASTRUCTURE.  Requires oracle/_ref/libdarm_ref.so (``make -C oracle ref``,
built from /root/reference/proj/src).  Every number in the fixtures comes from the
reference's own code: makeRandomInput (fixtures.cpp:82-108), runDarm
(melding_driver.cpp:54-100) and executeWarp (interp.cpp:332-381) — see
DESIGN.md §Oracle.  Re-run with:

    python oracle/gen_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
POSITIVE = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested", "bitonic"]
WARPS = [1, 4, 8, 32, 64]
SEEDS = [1000, 1001, 3000, 5000]


def std_mt19937_64_kat():
    # C++ [rand.predef]: the 10000th invocation of a default-constructed
    # std::mt19937_64 (seed 5489) produces 9981545732273789042.
    return {"seed": 5489, "index": 10000, "value": 9981545732273789042}


def stats_rows(stats):
    keys = ["issuedInstructions", "threadCycles", "usefulThreadCycles", "serializedCycles",
            "divergentBranchCount", "sharedMemIssues", "globalMemIssues", "flags"]
    return [dict(zip(keys, map(int, row))) for row in stats]


def corpus_fixtures(ref: Reference, name: str) -> dict:
    orig = ref.load(name, 0)
    meld = ref.load(name, 1)
    sizes = [s for _, s in orig.globals]
    out = {
        "kernel": name,
        "params": orig.params,
        "globals": orig.globals,
        "shared": orig.shared,
        "melds": meld.layout["melds"],
        "cases": [],
    }

    def run_case(warp, seed, args_override=None, full_range=False):
        args, gl, sh = orig.make_random_input(warp, seed)
        if args_override is not None:
            args = np.array(args_override, dtype=np.int32)
        if full_range:
            rng = np.random.Generator(np.random.MT19937(seed))
            gl = rng.integers(-(2 ** 31), 2 ** 31, size=gl.size, dtype=np.int64).astype(np.int32)
        S = sizes[0]
        # one warp, full declared globals (gstride = declared size)
        gin = gl.copy()
        res = {}
        for tag, mod in (("unmelded", orig), ("melded", meld)):
            g = gin.copy()
            f, st = mod.execute_warps(warp, 1, args.reshape(-1, 1), g, S,
                                      shared=sh if orig.shared else None)
            _, st_unit = mod.execute_warps(warp, 1, args.reshape(-1, 1), gin.copy(), S,
                                           shared=sh if orig.shared else None, unit_latency=True)
            res[tag] = {"globals_final": g.tolist(), "faults": int(f[0]),
                        "stats": stats_rows(st)[0], "stats_unit_latency": stats_rows(st_unit)[0]}
        assert res["unmelded"]["globals_final"] == res["melded"]["globals_final"], (name, warp, seed)
        assert res["unmelded"]["faults"] == res["melded"]["faults"]
        case = {"warp": warp, "seed": seed, "args": args.tolist(), "full_range": full_range,
                "args_overridden": args_override is not None,
                "globals_init": gin.tolist(),
                "shared_init": sh.tolist() if orig.shared else [],
                "globals_final": res["unmelded"]["globals_final"],
                "faults": res["unmelded"]["faults"],
                "stats": {k: {"default": v["stats"], "unit": v["stats_unit_latency"]} for k, v in res.items()}}
        out["cases"].append(case)

    for warp in WARPS:
        for seed in SEEDS:
            run_case(warp, seed)
    # half-warp split (acceptance.cpp:248-258): n=16, or h=16,q=24
    if name != "bitonic":
        half = [16] if len(orig.params) == 1 else [16, 24]
        for seed in range(3000, 3010):
            run_case(32, seed, args_override=half)
        run_case(32, 7, args_override=half, full_range=True)
        run_case(64, 8, args_override=[40] if len(orig.params) == 1 else [20, 50], full_range=True)
    else:
        # every (k, dir) the sort visits at warp 32 and 64, plus k = warp (partner past the lanes)
        for warp in (32, 64):
            for dir_ in (2, 4, 8, 16, 32, 64):
                k = dir_ // 2
                while k >= 1:
                    run_case(warp, 6000 + dir_ * 100 + k, args_override=[k, dir_])
                    k //= 2
            run_case(warp, 7000, args_override=[warp, 2])      # k == warp: lanes read beyond
    return out


def bitonic_sort_fixtures(ref: Reference) -> dict:
    mod = ref.load("bitonic", 0)
    meld = ref.load("bitonic", 1)
    out = {"kernel": "bitonic", "cases": []}
    rng = np.random.Generator(np.random.MT19937(11))
    for B in (2, 4, 8, 16, 32, 64):
        for dup in (False, True):
            nb = 4
            if dup:
                keys = rng.integers(-128, 129, size=nb * B, dtype=np.int64).astype(np.int32)
            else:
                keys = rng.integers(-(2 ** 31), 2 ** 31, size=nb * B, dtype=np.int64).astype(np.int32)
            a = keys.copy()
            st_u = mod.bitonic_sort(a, B, unit_latency=True)
            b = keys.copy()
            st_m = meld.bitonic_sort(b, B, unit_latency=True)
            assert (a == b).all()
            assert (a.reshape(-1, B) == np.sort(keys.reshape(-1, B), axis=1)).all()
            out["cases"].append({"bucket": B, "keys": keys.tolist(), "sorted": a.tolist(),
                                 "stats_unit_latency": {"unmelded": st_u.tolist(), "melded": st_m.tolist()}})
    return out


OE_IR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2107_05681_b200", "ir", "oddeven_step.ir")


def oddeven_sort_fixtures(ref: Reference) -> dict:
    """PCM: the reference interpreter chains ir/oddeven_step.ir (original and
    as melded by runDarm) over every Batcher odd-even merge step of B-key
    buckets: sorted outputs and the simulator statistics (unit and default
    latencies: issued, threadCycles, usefulThreadCycles, serializedCycles,
    divergentBranchCount, sharedMemIssues, globalMemIssues)."""
    from oracle import oddeven_schedule

    text = open(OE_IR).read()
    mod = ref.load_text(text, 0)
    meld = ref.load_text(text, 1)
    out = {"ir": "paper_2107_05681_b200/ir/oddeven_step.ir", "melds": meld.layout["melds"], "cases": []}
    rng = np.random.Generator(np.random.MT19937(13))
    for B in (2, 4, 8, 16, 32, 64):
        for dup in (False, True):
            nb = 4
            lo, hi = (-128, 129) if dup else (-(2 ** 31), 2 ** 31)
            keys = rng.integers(lo, hi, size=nb * B, dtype=np.int64).astype(np.int32)
            a = keys.copy()
            st_u = mod.chain_sort(a, B, oddeven_schedule(B), unit_latency=True)
            b = keys.copy()
            st_m = meld.chain_sort(b, B, oddeven_schedule(B), unit_latency=True)
            assert (a == b).all()
            assert (a.reshape(-1, B) == np.sort(keys.reshape(-1, B), axis=1)).all()
            c, d = keys.copy(), keys.copy()
            dl_u = mod.chain_sort(c, B, oddeven_schedule(B))
            dl_m = meld.chain_sort(d, B, oddeven_schedule(B))
            assert (c == a).all() and (d == a).all()
            out["cases"].append({"bucket": B, "keys": keys.tolist(), "sorted": a.tolist(),
                                 "stats_unit_latency": {"unmelded": st_u.tolist(), "melded": st_m.tolist()},
                                 "stats_default_latency": {"unmelded": dl_u.tolist(), "melded": dl_m.tolist()}})
    return out


MS_IR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2107_05681_b200", "ir", "merge_step.ir")


def _merge_path(a, na, b, nb, d):
    lo, hi = max(0, d - nb), min(d, na)
    while lo < hi:
        mid = (lo + hi) // 2
        if a[mid] <= b[d - 1 - mid]:
            lo = mid + 1
        else:
            hi = mid
    return lo


def merge_chain(mod, keys, warp=32, chunk=16):
    """Bottom-up merge sort of keys (n <= 1024) by the reference interpreter:
    per pass, every merge is cut into `chunk`-output jobs (the host finds each
    job's start on the merge path, as the GPU does), jobs are dealt to the
    lanes of a warp, and ir/merge_step.ir runs to a fixpoint per batch."""
    n = len(keys)
    cur = np.zeros(1024, np.int32)
    cur[:n] = keys
    stats = np.zeros(7, np.int64)
    rounds = 0
    w = 1
    while w < n:
        jobs = []
        for a in range(0, n, 2 * w):
            iend, jend = min(a + w, n), min(a + 2 * w, n)
            A, B = cur[a:iend], cur[iend:jend]
            for s in range(0, jend - a, chunk):
                x = _merge_path(A, len(A), B, len(B), s)
                jobs.append((a + x, iend, iend + s - x, jend, a + s, min(a + s + chunk, jend)))
        dst = cur.copy()
        for b0 in range(0, len(jobs), warp):
            g = np.zeros(2 * 1024 + 6 * 64, np.int32)
            g[:1024] = cur
            g[1024:2048] = dst
            for t, (i, ie, j, je, k, ke) in enumerate(jobs[b0:b0 + warp]):
                for f, v in enumerate((i, j, k, ie, je, ke)):
                    g[2048 + 64 * f + t] = v
            r, st = mod.run_to_fixpoint(warp, np.zeros(0, np.int32), g, np.zeros(0, np.int32), unit_latency=True)
            rounds += r
            stats += st
            dst = g[1024:2048].copy()
        cur = dst
        w *= 2
    return cur[:n].copy(), stats, rounds


def merge_sort_fixtures(ref: Reference) -> dict:
    text = open(MS_IR).read()
    mod = ref.load_text(text, 0)
    meld = ref.load_text(text, 1)
    out = {"ir": "paper_2107_05681_b200/ir/merge_step.ir", "melds": meld.layout["melds"], "cases": []}
    rng = np.random.Generator(np.random.MT19937(17))
    for n in (1, 2, 3, 17, 64, 100, 256, 777, 1024):
        for dup in (False, True):
            lo, hi = (-8, 9) if dup else (-(2 ** 31), 2 ** 31)
            keys = rng.integers(lo, hi, size=n, dtype=np.int64).astype(np.int32)
            a, st_u, _ = merge_chain(mod, keys)
            b, st_m, _ = merge_chain(meld, keys)
            assert (a == b).all() and (a == np.sort(keys)).all(), (n, dup)
            out["cases"].append({"n": n, "keys": keys.tolist(), "sorted": a.tolist(),
                                 "stats_unit_latency": {"unmelded": st_u.tolist(), "melded": st_m.tolist()}})
    return out


NQ_IR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2107_05681_b200", "ir", "nqueens_sym.ir")


def nq_prefixes(n, base):
    out, mask = [], (1 << n) - 1

    def rec(row, cols, d1, d2):
        if row == base:
            out.append((cols, d1 & 0xFFFFFFFF, d2))
            return
        av = ~(cols | d1 | d2) & mask
        while av:
            b = av & -av
            av ^= b
            rec(row + 1, cols | b, ((d1 | b) << 1) & 0xFFFFFFFF, (d2 | b) >> 1)

    rec(0, 0, 0, 0)
    return out


def nqueens_chain_fixtures(ref: Reference) -> dict:
    """The reference interpreter runs ir/nqueens_sym.ir (original and as melded
    by runDarm) to a fixpoint per warp of prefixes: per-prefix solution counts
    and unit-latency utilisation.  The IR keeps the diagonals in board
    coordinates: st_d1 = d2_rel << base (bit r + c), st_d2 = (d1_rel & mask) <<
    (n - 1 - base) (bit c - r + n - 1)."""
    text = open(NQ_IR).read()
    orig = ref.load_text(text, 0)
    meld = ref.load_text(text, 1)
    out = {"ir": "paper_2107_05681_b200/ir/nqueens_sym.ir", "melds": meld.layout["melds"], "cases": []}
    W = 32
    for n, base in ((4, 1), (5, 1), (6, 2), (7, 2), (8, 2), (9, 2), (10, 3)):
        pre = nq_prefixes(n, base)
        mask = (1 << n) - 1
        case = {"n": n, "base": base, "prefixes": [list(p) for p in pre], "per_prefix": [],
                "stats_unit_latency": {"unmelded": [0] * 7, "melded": [0] * 7}, "rounds": {"unmelded": 0, "melded": 0}}
        for w0 in range(0, len(pre), W):
            chunk = pre[w0:w0 + W]
            res = {}
            for tag, mod in (("unmelded", orig), ("melded", meld)):
                g = np.zeros(6 * 64, np.int32)
                for t in range(W):
                    if t < len(chunk):
                        c, d1, d2 = chunk[t]
                        a1 = (d2 << base) & 0xFFFFFFFF
                        a2 = ((d1 & mask) << (n - 1 - base)) & 0xFFFFFFFF
                        g[t], g[64 + t] = base, c
                        g[128 + t], g[192 + t] = np.int64(a1).astype(np.int32), np.int64(a2).astype(np.int32)
                        g[256 + t] = ~(c | d1 | d2) & mask
                    else:
                        g[t] = base - 1
                sh = np.zeros(1024, np.int32)
                rounds, st = mod.run_to_fixpoint(W, np.array([n, mask, base], np.int32), g, sh, unit_latency=True)
                res[tag] = g[320:320 + len(chunk)].tolist()
                case["rounds"][tag] += rounds
                case["stats_unit_latency"][tag] = [a + int(b) for a, b in zip(case["stats_unit_latency"][tag], st)]
            assert res["unmelded"] == res["melded"], (n, base, w0)
            case["per_prefix"] += res["unmelded"]
        case["solutions"] = sum(case["per_prefix"])
        out["cases"].append(case)
    return out


NQ_STEP_IR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "paper_2107_05681_b200", "ir", "nqueens_step.ir")


def nqueens_step_chain_fixtures(ref: Reference) -> dict:
    """The paper-shaped encoding, ir/nqueens_step.ir (pop / count a leaf / push,
    an if-then-elseif-then that runDarm melds by region replication), run by
    the reference interpreter to a fixpoint per warp of prefixes, original and
    melded: per-prefix solution counts and unit-latency statistics.  Row-
    relative diagonals, as the host enumerates them."""
    text = open(NQ_STEP_IR).read()
    orig = ref.load_text(text, 0)
    meld = ref.load_text(text, 1)
    out = {"ir": "paper_2107_05681_b200/ir/nqueens_step.ir", "melds": meld.layout["melds"], "cases": []}
    W = 32
    for n, base in ((4, 1), (5, 1), (6, 2), (7, 2), (8, 2), (9, 2), (10, 3)):
        pre = nq_prefixes(n, base)
        mask = (1 << n) - 1
        case = {"n": n, "base": base, "per_prefix": [],
                "stats_unit_latency": {"unmelded": [0] * 7, "melded": [0] * 7}, "rounds": {"unmelded": 0, "melded": 0}}
        for w0 in range(0, len(pre), W):
            chunk = pre[w0:w0 + W]
            res = {}
            for tag, mod in (("unmelded", orig), ("melded", meld)):
                g = np.zeros(6 * 64, np.int32)
                for t in range(W):
                    if t < len(chunk):
                        c, d1, d2 = chunk[t]
                        g[t], g[64 + t] = base, c
                        g[128 + t], g[192 + t] = np.int64(d1).astype(np.int32), np.int64(d2).astype(np.int32)
                        g[256 + t] = ~(c | d1 | d2) & mask
                    else:
                        g[t] = base - 1
                sh = np.zeros(4 * 1024, np.int32)
                rounds, st = mod.run_to_fixpoint(W, np.array([n, mask, base], np.int32), g, sh, unit_latency=True)
                res[tag] = g[320:320 + len(chunk)].tolist()
                case["rounds"][tag] += rounds
                case["stats_unit_latency"][tag] = [a + int(b) for a, b in zip(case["stats_unit_latency"][tag], st)]
            assert res["unmelded"] == res["melded"], (n, base, w0)
            case["per_prefix"] += res["unmelded"]
        case["solutions"] = sum(case["per_prefix"])
        out["cases"].append(case)
    return out


def main():
    ref = Reference()
    os.makedirs(OUT, exist_ok=True)
    for name in POSITIVE:
        with open(os.path.join(OUT, f"corpus_{name}.json"), "w") as f:
            json.dump(corpus_fixtures(ref, name), f, separators=(",", ":"))
    with open(os.path.join(OUT, "bitonic_sort.json"), "w") as f:
        json.dump(bitonic_sort_fixtures(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "merge_sort.json"), "w") as f:
        json.dump(merge_sort_fixtures(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "oddeven_sort.json"), "w") as f:
        json.dump(oddeven_sort_fixtures(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "nqueens_chain.json"), "w") as f:
        json.dump(nqueens_chain_fixtures(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "nqueens_step_chain.json"), "w") as f:
        json.dump(nqueens_step_chain_fixtures(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "mt19937_64.json"), "w") as f:
        json.dump(std_mt19937_64_kat(), f)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
