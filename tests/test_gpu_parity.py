"""GPU parity: the sm_100a kernels against the reference oracle, bit-exact.

Every test calls through the C-ABI (libdarm_gpu.so) and compares with
* the golden vectors the unmodified reference produced (tests/golden/),
* the C restatement (oracle/darm_oracle.c) on large seeded batches, and
* when oracle/_ref is present, the reference itself with its own compareRuns.
"""
import numpy as np
import pytest

from conftest import CORPUS, load_golden

import paper_2107_05681_b200 as darm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def gpu():
    import torch

    assert torch.cuda.is_available(), "GPU tests need an sm_100 device"
    torch.cuda.set_device(0)
    darm.init()
    yield
    darm.shutdown() if hasattr(darm, "shutdown") else None


def _golden_batch(kernel):
    """Group the golden single-warp cases by warp size into compact batches."""
    gold = load_golden(f"corpus_{kernel}.json")
    S = gold["globals"][0][1]
    names = [n for n, _ in gold["globals"]]
    by_warp = {}
    for case in gold["cases"]:
        by_warp.setdefault(case["warp"], []).append(case)
    for W, cases in sorted(by_warp.items()):
        nw = len(cases)
        args = np.array([c["args"] for c in cases], dtype=np.int32).T.copy()
        g_in = {n: np.concatenate([np.array(c["globals_init"][i * S:i * S + W], np.int32) for c in cases])
                for i, n in enumerate(names)}
        g_out = {n: np.concatenate([np.array(c["globals_final"][i * S:i * S + W], np.int32) for c in cases])
                 for i, n in enumerate(names)}
        shared = None
        if gold["shared"]:
            shared = {"buf": np.concatenate([np.array(c["shared_init"], np.int32) for c in cases])}
        faults = np.array([c["faults"] for c in cases], np.int32)
        yield W, nw, args, g_in, g_out, shared, faults


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("kernel", CORPUS)
def test_golden_vectors(kernel, variant):
    for W, nw, args, g_in, g_out, shared, faults in _golden_batch(kernel):
        g = {n: v.copy() for n, v in g_in.items()}
        res = darm.execute_warps(kernel, variant, W, args, g, shared, n_warps=nw)
        for n in g_out:
            assert (res.globals[n] == g_out[n]).all(), (kernel, variant, W, n)
        assert (res.faults == faults).all(), (kernel, variant, W)


def _random_batch(kernel, warp, nw, seed, mode):
    info = darm.kernel_info(kernel)
    rng = np.random.default_rng(seed)
    names = [n for n, _ in info["globals"]]
    g = {n: rng.integers(-(2 ** 31), 2 ** 31, size=nw * warp, dtype=np.int64).astype(np.int32) for n in names}
    shared = None
    if kernel == "bitonic":
        acount = {"broadcast": 1, "warp": nw, "lane": nw * warp}[mode]
        ks = 1 << rng.integers(0, 7, size=acount)
        args = np.stack([ks, rng.integers(0, 2 * warp, size=acount)]).astype(np.int32)
        shared = {"buf": rng.integers(-(2 ** 31), 2 ** 31, size=nw * 64, dtype=np.int64).astype(np.int32)}
    else:
        acount = {"broadcast": 1, "warp": nw, "lane": nw * warp}[mode]
        args = rng.integers(-2, warp + 3, size=(len(info["params"]), acount)).astype(np.int32)
    return names, g, args, shared


@pytest.mark.parametrize("mode", ["broadcast", "warp", "lane"])
@pytest.mark.parametrize("kernel", CORPUS)
def test_random_batches_vs_restatement(kernel, mode, restatement):
    for warp in (1, 5, 32, 64):
        nw = 4096 if warp < 32 else 1024
        names, g, args, shared = _random_batch(kernel, warp, nw, 100 + warp, mode)
        want = np.concatenate([g[n] for n in names])
        wf = restatement.execute_warps(kernel, warp, nw, args, want, warp,
                                       None if shared is None else shared["buf"])
        for variant in (0, 1, 2):
            gg = {n: v.copy() for n, v in g.items()}
            res = darm.execute_warps(kernel, variant, warp, args, gg, shared, n_warps=nw)
            got = np.concatenate([res.globals[n] for n in names])
            assert (got == want).all(), (kernel, variant, warp, mode)
            assert (res.faults == wf).all(), (kernel, variant, warp, mode)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_sb1_config1_million_lanes_vs_reference(variant, restatement, reference):
    """BASELINE config 1: 2^20 int32 lanes = 32,768 warps of makeRandomInput
    fixtures with the half-warp split n=16, checked against the reference's
    executeWarp + compareRuns on every warp slice."""
    nw = 1 << 15
    batch = darm.make_random_input("sb1", 32, nw, 1000)
    names = ["in", "aux2", "aux3", "out"]
    g0 = np.concatenate([batch.globals[n] for n in names])
    mod = reference.load("sb1", int(variant == 1))
    ref = g0.copy()
    fr, _ = mod.execute_warps(32, nw, np.array([[16]], np.int32), ref, 32, None, threads=8, want_stats=False)
    g = {n: batch.globals[n].copy() for n in names}
    res = darm.execute_warps("sb1", variant, 32, [[16]], g)
    got = np.concatenate([res.globals[n] for n in names])
    w, diff = reference.compare_warps(mod, 32, nw, 32, ref, fr, got, res.faults)
    assert w == -1, (w, diff)
    # per-warp n from the fixtures themselves (makeRandomInput's %n)
    g = {n: batch.globals[n].copy() for n in names}
    res = darm.execute_warps("sb1", variant, 32, batch.args, g)
    want = g0.copy()
    restatement.execute_warps("sb1", 32, nw, batch.args, want, 32)
    assert (np.concatenate([res.globals[n] for n in names]) == want).all()


@pytest.mark.parametrize("kernel", CORPUS)
def test_device_mode_matches_host_mode(kernel):
    import torch

    names, g, args, shared = _random_batch(kernel, 32, 2048, 7, "warp")
    for variant in (0, 1, 2):
        host = {n: v.copy() for n, v in g.items()}
        rh = darm.execute_warps(kernel, variant, 32, args, host, shared, n_warps=2048)
        dev = {n: torch.from_numpy(v.copy()).cuda() for n, v in g.items()}
        dsh = {k: torch.from_numpy(v).cuda() for k, v in shared.items()} if shared else None
        rd = darm.execute_warps(kernel, variant, 32, torch.from_numpy(args).cuda(), dev, dsh, n_warps=2048)
        torch.cuda.synchronize()
        for n in names:
            assert (rd.globals[n].cpu().numpy() == rh.globals[n]).all()
        assert (rd.faults.cpu().numpy() == rh.faults).all()


@pytest.mark.parametrize("kpt", [0, 1, 4, 8, 16])
def test_bitonic_sort_golden(kpt):
    gold = load_golden("bitonic_sort.json")
    for case in gold["cases"]:
        B = case["bucket"]
        if kpt > 1 and (kpt > B or B // kpt > 32):
            continue
        for variant in (0, 1, 2, 3):
            keys = np.array(case["keys"], dtype=np.int32)
            st = darm.bitonic_sort(keys, B, variant, keys_per_thread=kpt)
            assert keys.tolist() == case["sorted"], (B, variant, kpt)
            if kpt:
                assert st["keys_per_thread"] == kpt


BUCKET_KPT = [(B, r) for B in (4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096) for r in (4, 8, 16)
              if r <= B and B // r <= 256]


@pytest.mark.parametrize("bucket,kpt", BUCKET_KPT)
def test_bitonic_sort_register_blocked(bucket, kpt):
    """Register-blocked forms (kpt keys per thread) against np.sort: full-range
    and duplicate-heavy keys, a ragged tail (n not a multiple of the 32*kpt
    warp tile) and a size that leaves most warps idle."""
    import torch

    rng = np.random.default_rng(bucket * 100 + kpt)
    for n in (1 << 18, bucket * 37, bucket):
        for dup in (False, True):
            lo, hi = (-128, 129) if dup else (-(2 ** 31), 2 ** 31)
            keys = rng.integers(lo, hi, size=n, dtype=np.int64).astype(np.int32)
            want = np.sort(keys.reshape(-1, bucket), axis=1).reshape(-1)
            for variant in (0, 1, 2, 3):
                k = torch.from_numpy(keys.copy()).cuda()
                st = darm.bitonic_sort(k, bucket, variant, keys_per_thread=kpt)
                assert st["keys_per_thread"] == kpt
                assert (k.cpu().numpy() == want).all(), (bucket, kpt, n, dup, variant)


@pytest.mark.parametrize("sort", ["bitonic", "oddeven"])
@pytest.mark.parametrize("kpt", [8, 16])
def test_register_sorts_16_byte_aligned_keys(sort, kpt):
    """The register-blocked kernels move keys as 32-byte vectors when the key
    pointer is 32-byte aligned and as 16-byte vectors otherwise: a pointer 16
    bytes past a 256-byte allocation takes the second path; both agree with
    np.sort (and a tail of partial CTA tiles)."""
    import torch

    fn = darm.bitonic_sort if sort == "bitonic" else darm.oddeven_sort
    rng = np.random.default_rng(kpt)
    for bucket in (64, 256):
        n = bucket * 1031
        keys = rng.integers(-(2 ** 31), 2 ** 31, size=n, dtype=np.int64).astype(np.int32)
        want = np.sort(keys.reshape(-1, bucket), axis=1).reshape(-1)
        for variant in ((0, 1, 2, 3) if sort == "bitonic" else (0, 1, 2)):
            buf = torch.zeros(n + 4, dtype=torch.int32, device="cuda")
            k = buf[4:]
            assert k.data_ptr() % 32 == 16
            k.copy_(torch.from_numpy(keys))
            assert fn(k, bucket, variant, keys_per_thread=kpt)["keys_per_thread"] == kpt
            assert (k.cpu().numpy() == want).all(), (sort, bucket, kpt, variant)
            assert (buf[:4].cpu().numpy() == 0).all()


def test_bitonic_sort_keys_per_thread_contract():
    import torch

    buf = torch.zeros(64 * 4 + 1, dtype=torch.int32, device="cuda")
    mis = buf[1:]                      # 4-byte aligned only
    with pytest.raises(darm.DarmError):
        darm.bitonic_sort(mis, 64, 1, keys_per_thread=16)
    assert darm.bitonic_sort(mis, 64, 1)["keys_per_thread"] == 1   # auto falls back
    with pytest.raises(darm.DarmError):
        darm.bitonic_sort(buf[:64 * 4], 64, 1, keys_per_thread=2)
    with pytest.raises(darm.DarmError):
        darm.bitonic_sort(buf[:64 * 3], 128, 1, keys_per_thread=16)   # n not a multiple of the bucket
    big = torch.zeros(8192, dtype=torch.int32, device="cuda")
    with pytest.raises(darm.DarmError):
        darm.bitonic_sort(big, 4096, 1, keys_per_thread=8)            # 512 threads per bucket
    with pytest.raises(darm.DarmError):
        darm.bitonic_sort(big, 2048, 1, keys_per_thread=1)            # one key per thread: bucket <= 1024
    with pytest.raises(darm.DarmError):
        darm.bitonic_sort(big, 8192, 1)
    with pytest.raises(darm.DarmError):
        darm.oddeven_sort(big, 2048, 1)                               # PCM: bucket <= 1024
    assert darm.oddeven_sort(big[:4096], 1024, 1)["keys_per_thread"] == 1
    assert darm.bitonic_sort(big, 4096, 1)["keys_per_thread"] == 16
    assert darm.bitonic_sort(buf[:64 * 4], 64, 1)["keys_per_thread"] == 16


@pytest.mark.parametrize("bucket", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_bitonic_sort_buckets(bucket, restatement):
    rng = np.random.default_rng(bucket)
    n = 1 << 20
    for dup in (False, True):
        if dup:
            keys = rng.integers(-128, 129, size=n, dtype=np.int64).astype(np.int32)
        else:
            keys = rng.integers(-(2 ** 31), 2 ** 31, size=n, dtype=np.int64).astype(np.int32)
        want = np.sort(keys.reshape(-1, bucket), axis=1).reshape(-1)
        chain = keys.copy()
        restatement.bitonic_sort(chain, bucket)
        assert (chain == want).all()
        for variant in (0, 1, 2, 3):
            k = keys.copy()
            darm.bitonic_sort(k, bucket, variant)
            assert (k == want).all(), (bucket, dup, variant)
    # ragged tail: n not a multiple of the CTA tile
    k = rng.integers(-(2 ** 31), 2 ** 31, size=bucket * 3, dtype=np.int64).astype(np.int32)
    want = np.sort(k.reshape(-1, bucket), axis=1).reshape(-1)
    darm.bitonic_sort(k, bucket, 1)
    assert (k == want).all()


@pytest.mark.parametrize("bucket", [64, 4096])
def test_bitonic_sort_host_pipeline(bucket):
    """HOST mode at 2^22 keys: 2^21-key chunks pipelined over three streams
    (copy in / sort / copy out); every bucket sorted, both forms, including
    4096-key buckets whose strides cross warps."""
    rng = np.random.default_rng(bucket)
    keys = rng.integers(-(2 ** 31), 2 ** 31, size=1 << 22, dtype=np.int64).astype(np.int32)
    want = np.sort(keys.reshape(-1, bucket), axis=1).reshape(-1)
    for variant in (0, 1, 2, 3):
        k = keys.copy()
        st = darm.bitonic_sort(k, bucket, variant)
        assert st["launches"] == 2 and st["keys_per_thread"] == 16
        assert (k == want).all(), (bucket, variant)


def test_bitonic_sort_config2_full_size():
    """BASELINE config 2: 2^24 int32 keys on one GPU, 64-key buckets; the
    size-independent properties: every bucket sorted and a permutation of its input."""
    import torch

    n = 1 << 24
    gen = torch.Generator(device="cuda").manual_seed(1)
    keys = torch.randint(-(2 ** 31), 2 ** 31 - 1, (n,), dtype=torch.int32, device="cuda", generator=gen)
    orig = keys.clone()
    for variant in (0, 1, 2, 3):
        k = orig.clone()
        darm.bitonic_sort(k, 64, variant)
        torch.cuda.synchronize()
        b = k.view(-1, 64)
        assert bool((b[:, 1:] >= b[:, :-1]).all())
        assert torch.equal(torch.sort(orig.view(-1, 64), dim=1).values, b)


def test_empty_inputs():
    keys = np.zeros(0, np.int32)
    darm.bitonic_sort(keys, 64, 1)
    g = {n: np.zeros(0, np.int32) for n in ["in", "aux2", "aux3", "out"]}
    res = darm.execute_warps("sb1", 1, 32, [[16]], g, n_warps=0)
    assert res.faults.size == 0
