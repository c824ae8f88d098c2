"""CPU-side checks of the C-ABI library (no GPU compute calls).

* libdarm_gpu.so loads and exports every function include/darm_gpu.h declares;
* kernel metadata mirrors the corpus declarations (pinned by the golden files);
* the host-side fixture generator reproduces makeRandomInput bit-exactly;
* without a GPU every compute entry point fails loudly (no CPU fallback);
* the SASS keeps the two forms distinct.
"""
import functools
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import CORPUS, ROOT, load_golden

import paper_2107_05681_b200 as darm

HEADER = os.path.join(ROOT, "include", "darm_gpu.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(darm_gpu_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(darm.LIB_PATH)
    names = header_functions()
    assert set(names) == set(darm.ABI_SYMBOLS)
    for name in names:
        assert hasattr(lib, name), name
    assert darm.lib().darm_gpu_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", darm.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


@pytest.mark.parametrize("kernel", CORPUS)
def test_kernel_info_matches_corpus(kernel):
    gold = load_golden(f"corpus_{kernel}.json")
    info = darm.kernel_info(kernel)
    assert info["params"] == gold["params"]
    assert info["globals"] == gold["globals"]
    assert info["shared"] == gold["shared"]


def test_kernel_list():
    assert darm.kernel_list() == CORPUS
    with pytest.raises(darm.DarmUserError):
        darm.kernel_info("neg_uniform")


@pytest.mark.parametrize("kernel", CORPUS)
def test_make_random_input_bit_exact(kernel):
    gold = load_golden(f"corpus_{kernel}.json")
    S = gold["globals"][0][1]
    ng = len(gold["globals"])
    for case in gold["cases"]:
        if case["full_range"]:
            continue
        b = darm.make_random_input(kernel, case["warp"], 1, case["seed"], gstride=S)
        got = np.concatenate([b.globals[n] for n, _ in gold["globals"]])
        assert got.tolist() == case["globals_init"]
        if gold["shared"]:
            assert b.shared["buf"].tolist() == case["shared_init"]
        if not case["args_overridden"]:
            assert b.args[:, 0].tolist() == case["args"]
    # batched: warp w uses seed0 + w, compact layout keeps the first `warp` words
    b = darm.make_random_input(kernel, 32, 5, 1000)
    for w in range(5):
        one = darm.make_random_input(kernel, 32, 1, 1000 + w, gstride=S)
        for n, _ in gold["globals"]:
            assert (b.globals[n][w * 32:(w + 1) * 32] == one.globals[n][:32]).all()
        assert (b.args[:, w] == one.args[:, 0]).all()
    assert ng == len(b.globals)


def test_make_random_input_multithreaded_matches_restatement(restatement):
    b = darm.make_random_input("sb1", 32, 5000, 77)       # >= 4096 warps: threaded path
    for w in (0, 1, 2500, 4999):
        args, words = restatement.make_random_input(["n"], [64, 64, 64, 64], 32, 77 + w)
        assert b.args[0, w] == args[0]
        for i, n in enumerate(["in", "aux2", "aux3", "out"]):
            assert (b.globals[n][w * 32:(w + 1) * 32] == words[i * 64:i * 64 + 32]).all()


def test_user_errors_are_reported_before_device_use():
    g = {n: np.zeros(32, np.int32) for n in ["in", "aux2", "aux3", "out"]}
    with pytest.raises(darm.DarmUserError):
        darm.execute_warps("nope", 0, 32, [[1]], {"in": np.zeros(32, np.int32)})
    with pytest.raises(darm.DarmUserError):
        darm.execute_warps("sb1", 0, 65, [[1]], g, n_warps=1)
    with pytest.raises(darm.DarmUserError):
        darm.execute_warps("sb1", 0, 32, np.zeros((1, 3), np.int32), g, n_warps=1)
    with pytest.raises(darm.DarmUserError):
        darm.bitonic_sort(np.zeros(96, np.int32), 48)
    with pytest.raises(darm.DarmUserError):
        darm.bitonic_sort(np.zeros(100, np.int32), 64)


def test_wrapper_rejects_bad_buffers():
    """The Python wrappers check dtype, contiguity and size before any pointer
    crosses the C-ABI (the library cannot see a buffer's extent)."""
    with pytest.raises(darm.DarmUserError):
        darm.bitonic_sort(np.zeros(128, np.float32), 64)
    with pytest.raises(darm.DarmUserError):
        darm.bitonic_sort(np.zeros(256, np.int32)[::2], 64)
    with pytest.raises(darm.DarmUserError):
        darm.merge_sort(np.zeros(16, np.int64))
    g = {n: np.zeros(64, np.int32) for n in ["in", "aux2", "aux3", "out"]}
    g["aux3"] = np.zeros(32, np.int32)   # two warps need 64 words
    with pytest.raises(darm.DarmUserError):
        darm.execute_warps("sb1", 0, 32, [[16]], g, n_warps=2)
    with pytest.raises(darm.DarmUserError):
        darm.lud(np.zeros((32, 16), np.float32))


def _have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_have_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(darm.DarmInternalError):
        darm.init()
    g = {n: np.zeros(32, np.int32) for n in ["in", "aux2", "aux3", "out"]}
    with pytest.raises(darm.DarmInternalError):
        darm.execute_warps("sb1", 0, 32, [[16]], g)
    with pytest.raises(darm.DarmInternalError):
        darm.bitonic_sort(np.zeros(64, np.int32), 64)


@functools.lru_cache(maxsize=1)
def _all_sass():
    from tools.sass_dump import sass_functions

    return sass_functions(darm.LIB_PATH)


def _sass(pattern):
    funcs = _all_sass()
    hits = [(n, b) for n, b in funcs.items() if pattern in n]
    assert len(hits) == 1, (pattern, [n for n, _ in hits])
    return [ins for _, ins in hits[0][1]]


def _ops(ins):
    """Opcode of each SASS instruction (predicate guard stripped)."""
    return [i.split()[1] if i.startswith("@") else i.split()[0] for i in ins]


def _load_classes(ins):
    return sorted({op for op in _ops(ins) if op.startswith("LDG")})


# IR branch arms per corpus kernel (sb1.ir ... nested.ir): every arm leads
# with DARM_IPDOM in the unmelded form
_ARMS = {"Sb1": 2, "Sb1r": 2, "Sb2T<false>": 4, "Sb2T<true>": 4, "Sb3T<false>": 6, "Sb3T<true>": 6,
         "Sb4T<false>": 4, "Sb4T<true>": 4, "Nested": 6}


@pytest.mark.parametrize("kernel", sorted(_ARMS))
def test_sass_unmelded_corpus_keeps_ipdom_branches(kernel):
    """SURVEY §7 H1 / interp.cpp:298-306: the unmelded form runs every IR arm
    behind a real divergent branch that reconverges at the post-dominator
    (BSSY ... @P BRA ... BSYNC), never as ptxas-predicated runs; the
    predicated column (variant 2) is the same source with the if-conversion
    left to ptxas; all three forms load the read-only inputs with the same
    class (LDG.E.CONSTANT)."""
    un = _sass(f"corpus_lanes<darm_gpu::{kernel}, 0, 32, 0>")
    me = _sass(f"corpus_lanes<darm_gpu::{kernel}, 1, 32, 0>")
    pr = _sass(f"corpus_lanes<darm_gpu::{kernel}, 2, 32, 0>")
    ou, op = _ops(un), _ops(pr)
    assert ou.count("PMTRIG") == _ARMS[kernel]
    assert sum(o.startswith("BSSY") for o in ou) >= 1 and sum(o.startswith("BSYNC") for o in ou) >= 1
    # a conditional branch per divergent condbr (plus the grid-stride loop)
    assert sum(bool(re.match(r"@!?P\d+ BRA", i)) for i in un) >= 2
    # no arm instruction is predicated in the unmelded form (the one guard
    # left is the loop's exit test)
    assert sum(i.startswith("@") and "BRA" not in i and "EXIT" not in i for i in un) <= 1
    assert "PMTRIG" not in op and "PMTRIG" not in _ops(me)
    assert _load_classes(un) == _load_classes(me) == _load_classes(pr) == ["LDG.E.CONSTANT"]


def test_sass_unmelded_keeps_both_arms():
    un = _sass("corpus_lanes<darm_gpu::Sb1, 0, 32, 0>")
    me = _sass("corpus_lanes<darm_gpu::Sb1, 1, 32, 0>")
    pr = _sass("corpus_lanes<darm_gpu::Sb1, 2, 32, 0>")
    # unmelded / predicated: both arms load `in` and store `out` (two STG, four
    # LDG); melded: one hoisted load of `in`, two guarded aux loads, one store.
    for form in (un, pr):
        assert sum(o.startswith("STG") for o in _ops(form)) == 2
        assert sum(o.startswith("LDG") for o in _ops(form)) == 4
    assert sum(o.startswith("STG") for o in _ops(me)) == 1
    assert sum(o.startswith("LDG") for o in _ops(me)) == 3
    # ptxas if-converts the predicated column: its arms are guarded runs
    assert sum(i.startswith("@") and "LDG" in i for i in pr) == 4


@pytest.mark.parametrize("kern,steps,pred_bssy", [("bitonic_sort_kernel<{}, 64, 256, 2>", 21, 2),
                                                  ("oddeven_sort_kernel<{}, 64, 256>", 21, 21)])
def test_sass_one_key_sorts_keep_ipdom_branches(kern, steps, pred_bssy):
    """One key per thread: the unmelded network branches on the lane's role in
    every step (both arms fenced).  The predicated column is what ptxas does
    with the same source unfenced: the bitonic min/max pairs are if-converted
    (no branch in the network); the PCM step keeps its three-way region (the
    shared-memory loads sit inside the arms, oddeven_sort.cu:121-132), so only
    the nested data-dependent if-thens are if-converted."""
    un = _sass(kern.format(0))
    pr = _sass(kern.format(2))
    ou = _ops(un)
    assert ou.count("PMTRIG") >= steps
    assert sum(o.startswith("BSSY") for o in ou) >= steps
    assert sum(o.startswith("BSYNC") for o in ou) >= steps
    assert "PMTRIG" not in _ops(pr)
    assert sum(o.startswith("BSSY") for o in _ops(pr)) <= pred_bssy
    me = _sass(kern.format(1))
    assert sum(o.startswith("BSSY") for o in _ops(me)) <= 2      # no branch in the network
    assert _load_classes(un) == _load_classes(me) == _load_classes(pr)


def test_sass_bitonic_sort_forms():
    un = _sass("bitonic_sort_kernel<2, 64, 256, 2>")
    me = _sass("bitonic_sort_kernel<1, 64, 256, 2>")
    li = _sass("bitonic_sort_kernel<3, 64, 256, 2>")
    # Same partner reads in every form (20 shuffles + 1 shared exchange for
    # B=64); the predicated unmelded network issues both arms of every `up`
    # branch (complementary predicated min/max), the melded one a single
    # keep-predicated min/max per step.
    # (two tiles per iteration, U = 2)
    for form in (un, me, li, _sass("bitonic_sort_kernel<0, 64, 256, 2>")):
        assert sum("SHFL.BFLY" in i for i in form) == 2 * 20
        assert sum("BAR.SYNC" in i for i in form) == 1
    assert len(un) > 1.4 * len(me)
    assert sum("IMNMX" in i for i in un) >= 2 * 60
    assert sum("IMNMX" in i for i in me) < 0.75 * sum("IMNMX" in i for i in un)
    # melded order flips run on the FMA pipe (IMAD), not as LOP3
    assert sum(i.startswith("IMAD") and "MOV" not in i for i in me) >= 2 * 5
    # the literal App. A.2 form: the same single predicated min/max per step
    # as the melded form, chosen by keep == up computed per lane (no order
    # flips: fewer IMADs), and no branch in the network either
    imnmx = lambda ins: sum("IMNMX" in i for i in ins)  # noqa: E731
    assert abs(imnmx(li) - imnmx(me)) <= 4
    assert sum(o.startswith("IMAD") for o in _ops(li)) < sum(o.startswith("IMAD") for o in _ops(me))
    assert sum(o.startswith("BSSY") for o in _ops(li)) <= 2


def test_sass_register_blocked_forms():
    """16 keys per thread, B = 64: the unmelded form keeps a conditional branch
    around the arms of every thread-dependent step; the melded form has none
    in the network (its few are the tile loop and the bounds checks)."""
    for kern in ("bitonic_sort_reg_kernel<{}, 64, 16, true>", "oddeven_sort_reg_kernel<{}, 64, 16>"):
        un = _sass(kern.format(0))
        me = _sass(kern.format(1))
        assert sum("SHFL" in i for i in un) > 0 and sum("SHFL" in i for i in me) > 0
        condbra = lambda ins: sum(bool(re.match(r"@!?U?P\d+ BRA", i)) and "DIV" not in i for i in ins)  # noqa: E731
        assert condbra(un) > condbra(me), kern
        assert _ops(un).count("PMTRIG") > 0
