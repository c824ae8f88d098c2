"""ctypes access to the oracle libraries.  TEST INFRASTRUCTURE ONLY.

Two checkers live under oracle/ (DESIGN.md §Oracle):

* ``Restatement`` — oracle/build/libdarm_oracle.so, the C restatement of the
  reference's runtime path (darm_oracle.c).  Always buildable (plain gcc).
* ``Reference``   — oracle/_ref/libdarm_ref.so, the UNMODIFIED reference sources
  (/root/reference/proj/src/*.cpp) compiled by oracle/Makefile plus the batching
  shim oracle/ref_shim.cpp.  Present wherever it was built (it travels to the GPU
  box inside the repo snapshot; /root/reference itself does not).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module; the product never does.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from typing import Dict, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "build", "libdarm_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libdarm_ref.so")
REF_ROOT = "/root/reference/proj"

I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)
U8P = ctypes.POINTER(ctypes.c_uint8)


def _p(a: Optional[np.ndarray], t=I32P):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def build(ref: bool = False) -> None:
    targets = ["all"] + (["ref"] if ref and os.path.isdir(REF_ROOT) else [])
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True, capture_output=True)


# ------------------------------------------------------------------ restatement
class Restatement:
    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.oracle_mt64_seed.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.oracle_mt64_next.argtypes = [ctypes.c_void_p]
        L.oracle_mt64_next.restype = ctypes.c_uint64
        L.oracle_make_random_input.argtypes = [ctypes.c_int, U8P, ctypes.c_int, I64P, ctypes.c_int,
                                               ctypes.c_uint64, I32P, I32P]
        L.oracle_execute_warps.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int64, I32P,
                                           ctypes.c_int64, I32P, ctypes.c_int64, I32P, I32P]
        L.oracle_bitonic_sort.argtypes = [I32P, ctypes.c_int64, ctypes.c_int]
        L.oracle_oddeven_sort.argtypes = [I32P, ctypes.c_int64, ctypes.c_int]
        L.oracle_merge_sort.argtypes = [I32P, ctypes.c_int64]
        L.oracle_lud.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_int]
        L.oracle_srad.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_float, I32P, ctypes.c_int]
        U32P = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_nqueens_prefixes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, U32P,
                                              ctypes.c_int64]
        L.oracle_nqueens_prefixes.restype = ctypes.c_int64
        L.oracle_nqueens_prefixes_ex.argtypes = [ctypes.c_int] * 5 + [U32P, ctypes.c_int64]
        L.oracle_nqueens_prefixes_ex.restype = ctypes.c_int64
        L.oracle_nqueens_count.argtypes = [ctypes.c_int, ctypes.c_int, U32P, ctypes.c_int64, U32P,
                                           ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_nqueens_count.restype = ctypes.c_uint64
        self.lib = L

    def mt64(self, seed: int, count: int) -> List[int]:
        state = ctypes.create_string_buffer(312 * 8 + 16)
        self.lib.oracle_mt64_seed(state, seed)
        return [self.lib.oracle_mt64_next(state) for _ in range(count)]

    def make_random_input(self, params: List[str], mems: List[int], warp: int, seed: int):
        kinds = np.array([1 if p[:1] in ("j", "k") else 0 for p in params] or [0], dtype=np.uint8)
        sizes = np.array(mems or [0], dtype=np.int64)
        args = np.zeros(max(1, len(params)), dtype=np.int32)
        words = np.zeros(max(1, int(sum(mems))), dtype=np.int32)
        self.lib.oracle_make_random_input(len(params), _p(kinds, U8P), len(mems), _p(sizes, I64P), warp,
                                          seed, _p(args), _p(words))
        return args[: len(params)], words[: int(sum(mems))]

    def execute_warps(self, kernel: str, warp: int, n_warps: int, args: np.ndarray,
                      globals_concat: np.ndarray, gstride: int, shared: Optional[np.ndarray] = None):
        """Mutates ``globals_concat`` in place; returns per-warp fault counts."""
        args = np.ascontiguousarray(args, dtype=np.int32)
        faults = np.zeros(max(1, n_warps), dtype=np.int32)
        rc = self.lib.oracle_execute_warps(kernel.encode(), warp, n_warps, _p(args), args.shape[-1],
                                           _p(globals_concat), gstride,
                                           _p(None if shared is None else np.ascontiguousarray(shared, dtype=np.int32)),
                                           _p(faults))
        if rc:
            raise ValueError(f"oracle_execute_warps({kernel}) -> {rc}")
        return faults[:n_warps]

    def bitonic_sort(self, keys: np.ndarray, bucket: int) -> None:
        rc = self.lib.oracle_bitonic_sort(_p(keys), keys.size, bucket)
        if rc:
            raise ValueError("oracle_bitonic_sort: bad bucket")

    def merge_sort(self, keys: np.ndarray) -> None:
        rc = self.lib.oracle_merge_sort(_p(keys), keys.size)
        if rc:
            raise ValueError("oracle_merge_sort failed")

    def oddeven_sort(self, keys: np.ndarray, bucket: int) -> None:
        rc = self.lib.oracle_oddeven_sort(_p(keys), keys.size, bucket)
        if rc:
            raise ValueError("oracle_oddeven_sort: bad bucket")

    def lud(self, a: np.ndarray, threads: int = 0) -> None:
        """In-place blocked LU in csrc/lud.cu's operation order."""
        assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"] and a.shape[0] == a.shape[1]
        rc = self.lib.oracle_lud(a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), a.shape[0],
                                 threads or (os.cpu_count() or 1))
        if rc:
            raise ValueError("oracle_lud: n must be a multiple of 16")

    def srad(self, j: np.ndarray, iters: int, lam: float, roi, threads: int = 0) -> None:
        """In-place SRAD in csrc/srad.cu's operation order."""
        assert j.dtype == np.float32 and j.flags["C_CONTIGUOUS"] and j.ndim == 2
        r = np.ascontiguousarray(roi, dtype=np.int32)
        rc = self.lib.oracle_srad(j.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), j.shape[0], j.shape[1], iters,
                                  lam, _p(r), threads or (os.cpu_count() or 1))
        if rc:
            raise ValueError(f"oracle_srad -> {rc}")

    def nqueens_prefixes(self, n: int, base: int, rank: int = 0, world: int = 1, mirror: bool = False) -> np.ndarray:
        cnt = self.lib.oracle_nqueens_prefixes_ex(n, base, rank, world, int(mirror), None, 0)
        out = np.zeros(3 * max(1, cnt), dtype=np.uint32)
        self.lib.oracle_nqueens_prefixes_ex(n, base, rank, world, int(mirror),
                                            _p(out, ctypes.POINTER(ctypes.c_uint32)), cnt)
        return out[: 3 * cnt].reshape(-1, 3)

    def nqueens_count_threads(self, n: int, base: int, states: np.ndarray, threads: int = 0):
        """nqueens_count over contiguous chunks of `states` on `threads` host
        threads (ctypes releases the GIL) -> (solutions, nodes below the prefixes)."""
        from concurrent.futures import ThreadPoolExecutor

        threads = threads or (os.cpu_count() or 1)
        chunks = np.array_split(np.arange(len(states)), threads * 8)
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(lambda ix: self.nqueens_count(n, base, states[ix])[::2] if len(ix) else (0, 0),
                              chunks))
        return sum(r[0] for r in res), sum(r[1] for r in res)

    def nqueens_count(self, n: int, base: int, states: np.ndarray):
        """-> (total solutions, per-prefix counts, placements below the prefixes)."""
        states = np.ascontiguousarray(states, dtype=np.uint32)
        per = np.zeros(max(1, len(states)), dtype=np.uint32)
        nodes = ctypes.c_uint64(0)
        U32P = ctypes.POINTER(ctypes.c_uint32)
        tot = self.lib.oracle_nqueens_count(n, base, _p(states, U32P), len(states), _p(per, U32P),
                                            ctypes.byref(nodes))
        return int(tot), per[: len(states)], int(nodes.value)


# ------------------------------------------------------------------ reference
class RefModule:
    def __init__(self, ref: "Reference", handle: ctypes.c_void_p):
        self.ref, self.h = ref, handle
        buf = ctypes.create_string_buffer(1 << 16)
        ref.lib.ref_layout(self.h, buf, 1 << 16)
        self.layout = json.loads(buf.value.decode())

    def __del__(self):
        try:
            self.ref.lib.ref_free(self.h)
        except Exception:
            pass

    @property
    def params(self) -> List[str]:
        return self.layout["params"]

    @property
    def globals(self) -> List[list]:
        return self.layout["globals"]

    @property
    def shared(self) -> List[list]:
        return self.layout["shared"]

    def text(self) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        self.ref.lib.ref_print(self.h, buf, 1 << 16)
        return buf.value.decode()

    def make_random_input(self, warp: int, seed: int):
        args = np.zeros(max(1, len(self.params)), dtype=np.int32)
        gl = np.zeros(max(1, sum(s for _, s in self.globals)), dtype=np.int32)
        sh = np.zeros(max(1, sum(s for _, s in self.shared)), dtype=np.int32)
        self.ref.lib.ref_make_random_input(self.h, warp, seed, _p(args), _p(gl), _p(sh))
        return args[: len(self.params)], gl, sh

    def execute_warps(self, warp: int, n_warps: int, args: np.ndarray, globals_concat: np.ndarray,
                      gstride: int, shared: Optional[np.ndarray] = None, unit_latency: bool = False,
                      threads: int = 1, want_stats: bool = True, max_steps: int = 10_000_000):
        args = np.ascontiguousarray(args, dtype=np.int32)
        faults = np.zeros(max(1, n_warps), dtype=np.int32)
        stats = np.zeros((max(1, n_warps), 8), dtype=np.int64) if want_stats else None
        err = ctypes.create_string_buffer(512)
        rc = self.ref.lib.ref_execute_warps(
            self.h, warp, n_warps, _p(args), args.shape[-1], _p(globals_concat), gstride,
            _p(None if shared is None else np.ascontiguousarray(shared, dtype=np.int32)),
            int(unit_latency), max_steps, threads, None, None, _p(faults),
            _p(stats, I64P) if stats is not None else None, err, 512)
        if rc:
            raise RuntimeError(err.value.decode())
        return faults[:n_warps], (stats[:n_warps] if stats is not None else None)

    def bitonic_sort(self, keys: np.ndarray, bucket: int, threads: int = 1, unit_latency: bool = False):
        stats = np.zeros(7, dtype=np.int64)
        err = ctypes.create_string_buffer(512)
        rc = self.ref.lib.ref_bitonic_sort(self.h, _p(keys), keys.size, bucket, threads, int(unit_latency),
                                           _p(stats, I64P), err, 512)
        if rc:
            raise RuntimeError(err.value.decode())
        return stats


def oddeven_schedule(bucket: int) -> np.ndarray:
    """(p, k, n) params of every Batcher odd-even merge step of a bucket, in
    order: p = 1, 2, .., B/2 and k = p, p/2, .., 1 (ir/oddeven_step.ir)."""
    steps = []
    p = 1
    while p < bucket:
        k = p
        while k >= 1:
            steps.append((p, k, bucket))
            k //= 2
        p *= 2
    return np.array(steps, dtype=np.int32).reshape(-1, 3)


def _chain_sort(self, keys: np.ndarray, bucket: int, schedule: np.ndarray, threads: int = 1,
                unit_latency: bool = False):
    """executeWarp chained over a network step kernel's schedule, per bucket (in place)."""
    stats = np.zeros(7, dtype=np.int64)
    err = ctypes.create_string_buffer(512)
    sched = np.ascontiguousarray(schedule, dtype=np.int32)
    rc = self.ref.lib.ref_chain_sort(self.h, _p(keys), keys.size, bucket, _p(sched), sched.shape[0],
                                     sched.shape[1], threads, int(unit_latency), _p(stats, I64P), err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return stats


RefModule.chain_sort = _chain_sort


def _execute_program(self, warp, n_warps, args, globals_, shared=None, latency=None, max_steps=10_000_000,
                     threads=1):
    """executeWarp per warp in the GPU program layout (globals / shared in/out,
    n_warps x words); -> (returns, has_ret, faults, stats[n_warps, 8])."""
    args = np.ascontiguousarray(args, dtype=np.int32)
    acount = args.shape[-1] if args.size else 1
    rets = np.zeros(max(1, n_warps * warp), np.int32)
    has = np.zeros(max(1, n_warps * warp), np.uint8)
    faults = np.zeros(max(1, n_warps), np.int32)
    stats = np.zeros((max(1, n_warps), 8), np.int64)
    lat = None if latency is None else np.ascontiguousarray(latency, dtype=np.int64)
    err = ctypes.create_string_buffer(512)
    rc = self.ref.lib.ref_execute_program(self.h, warp, n_warps, _p(args), acount, _p(globals_), _p(shared),
                                          _p(lat, I64P), max_steps, threads, _p(rets), _p(has, U8P), _p(faults),
                                          _p(stats, I64P), err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return (rets[:n_warps * warp].reshape(n_warps, warp), has[:n_warps * warp].reshape(n_warps, warp),
            faults[:n_warps], stats[:n_warps])


RefModule.execute_program = _execute_program


def _run_to_fixpoint(self, warp, args, globals_full, shared_full, max_rounds=1_000_000, unit_latency=False):
    """executeWarp chained to a fixpoint on one warp (declared-size arrays, in/out)."""
    args = np.ascontiguousarray(args, dtype=np.int32)
    stats = np.zeros(7, dtype=np.int64)
    rounds = np.zeros(1, dtype=np.int64)
    err = ctypes.create_string_buffer(512)
    rc = self.ref.lib.ref_run_to_fixpoint(self.h, warp, _p(args), _p(globals_full), _p(shared_full), max_rounds,
                                          int(unit_latency), _p(stats, I64P), _p(rounds, I64P), err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return int(rounds[0]), stats


RefModule.run_to_fixpoint = _run_to_fixpoint


class Reference:
    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        L.ref_load.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_double, ctypes.POINTER(vp),
                               ctypes.c_char_p, ctypes.c_size_t]
        L.ref_load_corpus.argtypes = L.ref_load.argtypes
        L.ref_corpus_text.argtypes = [ctypes.c_char_p]
        L.ref_corpus_text.restype = ctypes.c_char_p
        L.ref_free.argtypes = [vp]
        L.ref_print.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_print.restype = ctypes.c_size_t
        L.ref_layout.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_layout.restype = ctypes.c_size_t
        L.ref_make_random_input.argtypes = [vp, ctypes.c_int, ctypes.c_uint64, I32P, I32P, I32P]
        L.ref_execute_warps.argtypes = [vp, ctypes.c_int, ctypes.c_int64, I32P, ctypes.c_int64, I32P,
                                        ctypes.c_int64, I32P, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                        I32P, U8P, I32P, I64P, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_compare_warps.argtypes = [vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, I32P, I32P, U8P,
                                        I32P, I32P, I32P, U8P, I32P, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_compare_warps.restype = ctypes.c_int64
        L.ref_bitonic_sort.argtypes = [vp, I32P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       I64P, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_run_to_fixpoint.argtypes = [vp, ctypes.c_int, I32P, I32P, I32P, ctypes.c_int64, ctypes.c_int,
                                          I64P, I64P, ctypes.c_char_p, ctypes.c_size_t]
        L.ref_execute_program.argtypes = [vp, ctypes.c_int, ctypes.c_int64, I32P, ctypes.c_int64, I32P, I32P, I64P,
                                          ctypes.c_int64, ctypes.c_int, I32P, U8P, I32P, I64P, ctypes.c_char_p,
                                          ctypes.c_size_t]
        L.ref_chain_sort.argtypes = [vp, I32P, ctypes.c_int64, ctypes.c_int, I32P, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, I64P, ctypes.c_char_p, ctypes.c_size_t]
        self.lib = L

    def load(self, name: str, meld: int = 0, threshold: float = 0.2) -> RefModule:
        h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_load_corpus(name.encode(), meld, threshold, ctypes.byref(h), err, 512)
        if rc:
            raise RuntimeError(err.value.decode())
        return RefModule(self, h)

    def load_text(self, text: str, meld: int = 0, threshold: float = 0.2) -> RefModule:
        h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(512)
        rc = self.lib.ref_load(text.encode(), meld, threshold, ctypes.byref(h), err, 512)
        if rc:
            raise RuntimeError(err.value.decode())
        return RefModule(self, h)

    def compare_warps(self, mod: RefModule, warp: int, n_warps: int, gstride: int,
                      globals_a: np.ndarray, faults_a: np.ndarray, globals_b: np.ndarray,
                      faults_b: np.ndarray):
        """The reference's own compareRuns per warp slice -> (first bad warp or -1, diff)."""
        diff = ctypes.create_string_buffer(512)
        w = self.lib.ref_compare_warps(mod.h, warp, n_warps, gstride, _p(globals_a), None, None,
                                       _p(np.ascontiguousarray(faults_a, dtype=np.int32)), _p(globals_b),
                                       None, None, _p(np.ascontiguousarray(faults_b, dtype=np.int32)),
                                       diff, 512)
        return int(w), diff.value.decode()


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)
