"""Every kernel family once per form at small sizes, HOST buffers, no torch —
the workload of tests/test_sanitizer.py (compute-sanitizer memcheck /
racecheck / synccheck over it):

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05681_b200 as darm  # noqa: E402

CORPUS = ["sb1", "sb1r", "sb2", "sb2r", "sb3", "sb3r", "sb4", "sb4r", "nested"]
DIAMOND = """global x[64]
global y[64]
fn d(%n) {
^e:
  %t = tid
  %c = icmp.lt %t %n
  condbr %c ^l ^r
^l:
  %a = load.global x %t
  store.global y %t %a
  br ^j
^r:
  %b = load.global y %t
  store.global x %t %b
  br ^j
^j:
  ret
}
"""


def main():
    darm.init()
    rng = np.random.default_rng(0)
    for k in CORPUS + ["bitonic"]:
        b = darm.make_random_input(k, 32, 64, 1)
        args = b.args if k == "bitonic" else ([[16]] if len(b.args) == 1 else [[16], [24]])
        for v in ((0, 1) if k == "bitonic" else (0, 1, 2)):
            g = {n: a.copy() for n, a in b.globals.items()}
            sh = {n: a.copy() for n, a in b.shared.items()} or None
            darm.execute_warps(k, v, 32, args, g, sh)
    for B, kpts in ((64, (16, 1)), (256, (16, 1)), (1024, (16, 1)), (4096, (16,))):
        keys = rng.integers(-(2 ** 31), 2 ** 31, size=8192 if B < 4096 else 4 * 4096, dtype=np.int64).astype(np.int32)
        for kpt in kpts:
            for v in (0, 1, 2, 3):
                k = keys.copy()
                darm.bitonic_sort(k, B, v, keys_per_thread=kpt)
                assert (k.reshape(-1, B) == np.sort(keys.reshape(-1, B), axis=1)).all()
            if B <= 256:
                for v in (0, 1, 2):
                    k = keys.copy()
                    darm.oddeven_sort(k, B, v, keys_per_thread=kpt)
                    assert (k.reshape(-1, B) == np.sort(keys.reshape(-1, B), axis=1)).all()
    # one key per thread with several 256-key tiles per CTA (the exchange
    # buffers reused across tiles): 2^19 keys = 2048 tiles over <= 1184 CTAs
    keys = rng.integers(-(2 ** 31), 2 ** 31, size=1 << 19, dtype=np.int64).astype(np.int32)
    for B in (64, 128):
        for v in (0, 1):
            k = keys.copy()
            darm.oddeven_sort(k, B, v, keys_per_thread=1)
            assert (k.reshape(-1, B) == np.sort(keys.reshape(-1, B), axis=1)).all()
            k = keys.copy()
            darm.bitonic_sort(k, B, v, keys_per_thread=1)
            assert (k.reshape(-1, B) == np.sort(keys.reshape(-1, B), axis=1)).all()
    keys = rng.integers(-(2 ** 31), 2 ** 31, size=3 * 8192 + 5, dtype=np.int64).astype(np.int32)
    for v in (0, 1):
        k = keys.copy()
        darm.merge_sort(k, v)
        assert (k == np.sort(keys)).all()
    for v in (0, 1):
        assert darm.nqueens(8, 3, v, want_stats=False)[0] == 92
        assert darm.nqueens(10, 4, v, want_stats=False, mirror=True)[0] == 724
        assert darm.nqueens(10, 4, v, want_stats=False, mirror=True, paper_shape=True)[0] == 724
    n = 256
    a0 = (rng.random((n, n), dtype=np.float32) + n * np.eye(n, dtype=np.float32)).astype(np.float32)
    for v in (0, 1):
        a = a0.copy()
        darm.lud(a, v)
    j0 = np.exp(rng.random((70, 300), dtype=np.float32)).astype(np.float32)
    for fast in (False, True):
        for v in (0, 1):
            j = j0.copy()
            darm.srad(j, 3, 0.5, (0, 40, 3, 250), v, fast=fast)
    prog = darm.Program(DIAMOND)
    g = rng.integers(-100, 100, size=(16, prog.global_words), dtype=np.int64).astype(np.int32)
    prog.execute_warps(32, np.array([[16]], np.int32), g, n_warps=16)
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
