"""Pin the CPU restatement (oracle/darm_oracle.c) to the reference.

Golden vectors in tests/golden/ were produced by oracle/gen_golden.py running the
unmodified reference (makeRandomInput, runDarm, executeWarp).  When the reference
library itself is built (oracle/_ref), the restatement is also compared against
it live on larger random batches with the reference's own compareRuns.
"""
import numpy as np
import pytest

from conftest import CORPUS, load_golden


def test_mt19937_64_known_answer(restatement):
    kat = load_golden("mt19937_64.json")
    vals = restatement.mt64(kat["seed"], kat["index"])
    assert vals[-1] == kat["value"]


@pytest.mark.parametrize("kernel", CORPUS)
def test_make_random_input_matches_reference(restatement, kernel):
    gold = load_golden(f"corpus_{kernel}.json")
    mems = [s for _, s in gold["globals"]] + [s for _, s in gold["shared"]]
    ng = sum(s for _, s in gold["globals"])
    checked = 0
    for case in gold["cases"]:
        args, words = restatement.make_random_input(gold["params"], mems, case["warp"], case["seed"])
        if not case["full_range"]:
            assert words[:ng].tolist() == case["globals_init"]
        assert words[ng:].tolist() == case["shared_init"]
        if not case["args_overridden"]:
            assert args.tolist() == case["args"]
            checked += 1
    assert checked > 0


@pytest.mark.parametrize("kernel", CORPUS)
def test_execute_warps_matches_reference_golden(restatement, kernel):
    gold = load_golden(f"corpus_{kernel}.json")
    sizes = [s for _, s in gold["globals"]]
    S = sizes[0]
    assert all(s == S for s in sizes)
    for case in gold["cases"]:
        g = np.array(case["globals_init"], dtype=np.int32)
        shared = np.array(case["shared_init"], dtype=np.int32) if case["shared_init"] else None
        f = restatement.execute_warps(kernel, case["warp"], 1, np.array(case["args"]).reshape(-1, 1), g, S, shared)
        assert g.tolist() == case["globals_final"], (kernel, case["warp"], case["seed"])
        assert int(f[0]) == case["faults"], (kernel, case["warp"], case["seed"])


def test_bitonic_sort_matches_reference_golden(restatement):
    gold = load_golden("bitonic_sort.json")
    for case in gold["cases"]:
        keys = np.array(case["keys"], dtype=np.int32)
        restatement.bitonic_sort(keys, case["bucket"])
        assert keys.tolist() == case["sorted"]


def test_bitonic_sort_restatement_sorts(restatement):
    rng = np.random.default_rng(3)
    for B in (2, 8, 64, 256, 1024):
        keys = rng.integers(-(2 ** 31), 2 ** 31, size=B * 16, dtype=np.int64).astype(np.int32)
        want = np.sort(keys.reshape(-1, B), axis=1).reshape(-1)
        restatement.bitonic_sort(keys, B)
        assert (keys == want).all()


def test_golden_melded_direction_matches_survey():
    """Unit-latency utilization rises after melding (acceptance C5 direction)."""
    for kernel in CORPUS:
        gold = load_golden(f"corpus_{kernel}.json")
        pre = post = 0.0
        n = 0
        for case in gold["cases"]:
            if case["warp"] != 32:
                continue
            su = case["stats"]["unmelded"]["unit"]
            sm = case["stats"]["melded"]["unit"]
            pre += su["usefulThreadCycles"] / su["threadCycles"]
            post += sm["usefulThreadCycles"] / sm["threadCycles"]
            n += 1
        assert n and post / n >= pre / n - 1e-9, kernel


@pytest.mark.parametrize("kernel", CORPUS)
def test_restatement_matches_live_reference(restatement, reference, kernel):
    """Random batches (full-range words, per-lane args) through both, compared
    with the reference's own compareRuns (interp.cpp:383-426)."""
    for variant in (0, 1):
        mod = reference.load(kernel, variant)
        rng = np.random.default_rng(17 + variant)
        for warp in (3, 32, 64):
            nw = 64
            ng = len(mod.globals)
            g0 = rng.integers(-(2 ** 31), 2 ** 31, size=ng * nw * warp, dtype=np.int64).astype(np.int32)
            if kernel == "bitonic":
                args = np.stack([1 << rng.integers(0, 7, size=nw), rng.integers(0, 2 * warp, size=nw)]).astype(np.int32)
                shared = rng.integers(-(2 ** 31), 2 ** 31, size=nw * 64, dtype=np.int64).astype(np.int32)
            else:
                args = rng.integers(-2, warp + 2, size=(len(mod.params), nw * warp)).astype(np.int32)
                shared = None
            a = g0.copy()
            fa, _ = mod.execute_warps(warp, nw, args, a, warp, shared, threads=4, want_stats=False)
            b = g0.copy()
            fb = restatement.execute_warps(kernel, warp, nw, args, b, warp, shared)
            w, diff = reference.compare_warps(mod, warp, nw, warp, a, fa, b, fb)
            assert w == -1, (kernel, variant, warp, w, diff)


# OEIS A000170
NQUEENS = {1: 1, 2: 0, 3: 0, 4: 2, 5: 10, 6: 4, 7: 40, 8: 92, 9: 352, 10: 724, 11: 2680, 12: 14200,
           13: 73712, 14: 365596, 15: 2279184, 16: 14772512}


def test_nqueens_restatement_matches_reference_chain(restatement):
    """Per-prefix solution counts of the reference interpreter running
    ir/nqueens_sym.ir (original and melded) to a fixpoint."""
    gold = load_golden("nqueens_chain.json")
    for case in gold["cases"]:
        states = restatement.nqueens_prefixes(case["n"], case["base"])
        assert states.tolist() == case["prefixes"]
        tot, per, _ = restatement.nqueens_count(case["n"], case["base"], states)
        assert per.tolist() == case["per_prefix"]
        assert tot == case["solutions"] == NQUEENS[case["n"]]


def test_nqueens_melded_spec_is_the_reference_pass_output():
    """The melded CUDA form mirrors runDarm's output for ir/nqueens_sym.ir: one
    block-block meld of ^pop and ^push, and the reference's
    own simulator sees fewer serialized cycles after it (the paper's
    direction)."""
    gold = load_golden("nqueens_chain.json")
    assert [(m["kind"], m["selectsInserted"], m["unpredicatedRuns"]) for m in gold["melds"]] == \
        [("block-block", 7, 6)]
    big = gold["cases"][-1]["stats_unit_latency"]
    # stats: issued, threadCycles, usefulThreadCycles, serializedCycles, divergentBranches, shared, global
    assert big["melded"][3] < big["unmelded"][3]
    assert big["melded"][2] / big["melded"][1] > big["unmelded"][2] / big["unmelded"][1]


def test_nqueens_paper_shape_chain_and_melds(restatement):
    """ir/nqueens_step.ir, the paper's shape (pop / count a leaf / push, an
    if-then-elseif-then): runDarm melds it by region
    replication — two block-region melds — and the reference
    interpreter running it (original and melded) to a fixpoint gives the
    restatement's per-prefix counts.  Its simulator sees higher utilisation
    after the meld but more issued instructions (the replicated region)."""
    gold = load_golden("nqueens_step_chain.json")
    assert [m["kind"] for m in gold["melds"]] == ["block-region", "block-region"]
    for case in gold["cases"]:
        states = restatement.nqueens_prefixes(case["n"], case["base"])
        tot, per, _ = restatement.nqueens_count(case["n"], case["base"], states)
        assert per.tolist() == case["per_prefix"]
        assert tot == case["solutions"] == NQUEENS[case["n"]]
    big = gold["cases"][-1]["stats_unit_latency"]
    assert big["melded"][2] / big["melded"][1] > big["unmelded"][2] / big["unmelded"][1]
    assert big["melded"][0] > big["unmelded"][0]


@pytest.mark.parametrize("n", range(4, 13))
def test_nqueens_restatement_known_answers(restatement, n):
    for base in (1, 2, n - 1):
        states = restatement.nqueens_prefixes(n, base)
        assert restatement.nqueens_count(n, base, states)[0] == NQUEENS[n]
    # rank partition covers every prefix exactly once
    parts = [restatement.nqueens_prefixes(n, 2, r, 3) for r in range(3)]
    assert sum(len(p) for p in parts) == len(restatement.nqueens_prefixes(n, 2))


def test_nqueens_node_count_n8(restatement):
    # nodes = root + placements of the prefix rows + placements below them
    states = restatement.nqueens_prefixes(8, 2)
    _, _, below = restatement.nqueens_count(8, 2, states)
    assert 1 + 8 + len(states) + below == 2057


def test_nqueens_prefix_count_matches_library(restatement):
    import paper_2107_05681_b200 as darm

    for n, base, rank, world in ((8, 2, 0, 1), (12, 3, 1, 4), (16, 6, 0, 1), (16, 6, 5, 8)):
        assert darm.lib().darm_gpu_nqueens_prefix_count(n, base, rank, world) == \
            len(restatement.nqueens_prefixes(n, base, rank, world))
