"""paper_2107_05681_b200 — B200-native runtime path for the DARM corpus kernels.

Python host side over the C-ABI in ``include/darm_gpu.h`` (``_lib/libdarm_gpu.so``,
sm_100a only).  The functions mirror the reference's runtime interface
(/root/reference/proj/include/darm/interp.hpp, fixtures.hpp):

=====================================  ==============================================
reference                              here
=====================================  ==============================================
``makeRandomInput`` fixtures.hpp:28     :func:`make_random_input` (n consecutive seeds)
``executeWarp``     interp.hpp:57       :func:`execute_warps` (a batch of warps)
``WarpResult.globalFinal/faults``       :class:`WarpBatchResult`
``compareRuns``     interp.hpp:67       :func:`compare_runs` (same verdict order)
corpus chain of ``bitonic.ir`` steps    :func:`bitonic_sort`
=====================================  ==============================================

Errors raise :class:`DarmUserError` (C-ABI code 2, the reference's
``std::runtime_error`` / CLI exit 2) or :class:`DarmInternalError` (code 3,
``std::logic_error`` / CUDA failures / CLI exit 3).  There is no CPU fallback:
if the shared library is missing or no sm_100 device is present, every compute
call raises.
"""
from __future__ import annotations

import ctypes
import functools
import json
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

UNMELDED = 0             # original CFG, every arm a real divergent branch (IPDOM)
MELDED = 1               # the control flow runDarm emits
PREDICATED = 2           # original CFG as ptxas compiles it (short arms if-converted)
MELDED_LITERAL = 3       # bitonic sorts: SURVEY App. A.2's select chain as printed
VARIANTS = {"unmelded": UNMELDED, "melded": MELDED, "predicated": PREDICATED, "melded_literal": MELDED_LITERAL}
FAST_MATH = 0x100   # SRAD: OR into the variant (DARM_FAST_MATH, within 1e-5 relative)
SRAD_ALL_ROWS, SRAD_INTERIOR_ROWS, SRAD_EDGE_ROWS = 0, 1, 2   # darm_gpu_srad_tile_step `part`

_HERE = os.path.dirname(os.path.abspath(__file__))
# DARM_GPU_LIB points experiments at a variant build (e.g. a knob sweep)
# without overwriting the in-tree library
LIB_PATH = os.environ.get("DARM_GPU_LIB") or os.path.join(_HERE, "_lib", "libdarm_gpu.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "darm_gpu.h")

# Every symbol include/darm_gpu.h declares.
ABI_SYMBOLS = (
    "darm_gpu_init",
    "darm_gpu_abi_version",
    "darm_gpu_shutdown",
    "darm_gpu_kernel_info",
    "darm_gpu_kernel_list",
    "darm_gpu_make_random_input",
    "darm_gpu_execute_warps",
    "darm_gpu_bitonic_sort",
    "darm_gpu_bitonic_sort_ex",
    "darm_gpu_oddeven_sort",
    "darm_gpu_merge_sort",
    "darm_gpu_nqueens",
    "darm_gpu_nqueens_prefix_count",
    "darm_gpu_nqueens_ex",
    "darm_gpu_nqueens_prefix_count_ex",
    "darm_gpu_lud",
    "darm_gpu_srad",
    "darm_gpu_srad_roi_words",
    "darm_gpu_srad_pitch",
    "darm_gpu_srad_tile_roi",
    "darm_gpu_srad_tile_step",
    "darm_gpu_srad_group_create",
    "darm_gpu_srad_group_connect",
    "darm_gpu_srad_group_load",
    "darm_gpu_srad_group_run",
    "darm_gpu_srad_group_read",
    "darm_gpu_srad_group_rows",
    "darm_gpu_srad_group_free",
    "darm_gpu_program_load",
    "darm_gpu_program_free",
    "darm_gpu_program_shape",
    "darm_gpu_program_memory",
    "darm_gpu_program_param",
    "darm_gpu_program_execute",
)


class DarmError(RuntimeError):
    code = 3


class DarmUserError(DarmError):
    code = 2


class DarmInternalError(DarmError):
    code = 3


class Stats(ctypes.Structure):
    _fields_ = [
        ("kernel_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("algorithmic_bytes", ctypes.c_uint64),
        ("launches", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}
        d["keys_per_thread"] = self.reserved  # call-specific; bitonic sort only
        return d


_lib = None


def lib() -> ctypes.CDLL:
    """Load libdarm_gpu.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DarmInternalError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(LIB_PATH)
        c_i32p = ctypes.POINTER(ctypes.c_int32)
        c_i32pp = ctypes.POINTER(c_i32p)
        L.darm_gpu_init.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_abi_version.restype = ctypes.c_int
        L.darm_gpu_shutdown.restype = None
        L.darm_gpu_kernel_info.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_kernel_info.restype = ctypes.c_size_t
        L.darm_gpu_kernel_list.restype = ctypes.c_char_p
        L.darm_gpu_make_random_input.argtypes = [
            ctypes.c_char_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, c_i32p, c_i32pp,
            ctypes.c_int64, c_i32pp, ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_execute_warps.argtypes = [
            ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, c_i32p, ctypes.c_int64,
            c_i32pp, ctypes.c_int, c_i32pp, ctypes.c_int, c_i32p, ctypes.c_int, ctypes.c_void_p,
            ctypes.POINTER(Stats), ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_bitonic_sort.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.POINTER(Stats), ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_bitonic_sort_ex.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.POINTER(Stats), ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_oddeven_sort.argtypes = L.darm_gpu_bitonic_sort_ex.argtypes
        vp = ctypes.c_void_p
        L.darm_gpu_program_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(vp),
                                            ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_program_free.argtypes = [vp]
        L.darm_gpu_program_free.restype = None
        L.darm_gpu_program_shape.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int)] * 3 + \
            [ctypes.POINTER(ctypes.c_int64)] * 2
        L.darm_gpu_program_memory.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                              ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]
        L.darm_gpu_program_memory.restype = ctypes.c_char_p
        L.darm_gpu_program_param.argtypes = [vp, ctypes.c_int]
        L.darm_gpu_program_param.restype = ctypes.c_char_p
        L.darm_gpu_program_execute.argtypes = [vp, ctypes.c_int, ctypes.c_int64, vp, ctypes.c_int64, vp, vp, vp, vp,
                                               vp, vp, ctypes.c_int64, ctypes.c_int, vp, ctypes.POINTER(Stats),
                                               ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_merge_sort.argtypes = [
            ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(Stats),
            ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_nqueens.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.POINTER(Stats), ctypes.c_char_p,
            ctypes.c_size_t]
        L.darm_gpu_nqueens_prefix_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.darm_gpu_nqueens_prefix_count.restype = ctypes.c_int64
        L.darm_gpu_nqueens_ex.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.POINTER(Stats), ctypes.c_char_p,
            ctypes.c_size_t]
        L.darm_gpu_nqueens_prefix_count_ex.argtypes = [ctypes.c_int] * 5
        L.darm_gpu_nqueens_prefix_count_ex.restype = ctypes.c_int64
        L.darm_gpu_lud.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.POINTER(Stats), ctypes.c_char_p, ctypes.c_size_t]
        I32P, F32P, F64P = c_i32p, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)
        L.darm_gpu_srad.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_float, I32P, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(Stats),
                                    ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_srad_roi_words.argtypes = [ctypes.c_int64, I32P]
        L.darm_gpu_srad_roi_words.restype = ctypes.c_int64
        L.darm_gpu_srad_pitch.argtypes = [ctypes.c_int64]
        L.darm_gpu_srad_pitch.restype = ctypes.c_int64
        L.darm_gpu_srad_tile_roi.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_int64, I32P, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_srad_tile_step.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_float, I32P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_int, ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
        VP, E = ctypes.c_void_p, [ctypes.c_char_p, ctypes.c_size_t]
        L.darm_gpu_srad_group_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_float, I32P,
                                                 ctypes.c_int, ctypes.c_int, ctypes.POINTER(VP), VP] + E
        L.darm_gpu_srad_group_connect.argtypes = [VP, VP] + E
        L.darm_gpu_srad_group_load.argtypes = [VP, VP, ctypes.c_int, VP] + E
        L.darm_gpu_srad_group_run.argtypes = [VP, ctypes.c_int, VP, ctypes.POINTER(Stats)] + E
        L.darm_gpu_srad_group_read.argtypes = [VP, VP, ctypes.c_int, VP] + E
        L.darm_gpu_srad_group_rows.argtypes = [VP, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.darm_gpu_srad_group_free.argtypes = [VP]
        L.darm_gpu_srad_group_free.restype = None
        _lib = L
    return _lib


def _check(rc: int, err: ctypes.Array) -> None:
    if rc == 0:
        return
    msg = err.value.decode(errors="replace")
    if rc == 2:
        raise DarmUserError(msg)
    raise DarmInternalError(msg or f"libdarm_gpu error {rc}")


def init() -> int:
    """Number of CUDA devices (raises DarmInternalError without an sm_100 GPU)."""
    n = ctypes.c_int(0)
    err = ctypes.create_string_buffer(512)
    _check(lib().darm_gpu_init(ctypes.byref(n), err, 512), err)
    return n.value


def kernel_list() -> List[str]:
    return lib().darm_gpu_kernel_list().decode().split(",")


@functools.lru_cache(maxsize=None)
def _kernel_info_json(kernel: str) -> str:
    buf = ctypes.create_string_buffer(4096)
    n = lib().darm_gpu_kernel_info(kernel.encode(), buf, 4096)
    if n == 0:
        raise DarmUserError(f"unknown kernel '{kernel}'")
    return buf.value.decode()


def kernel_info(kernel: str) -> dict:
    return json.loads(_kernel_info_json(kernel))


def _i32p(a: np.ndarray):
    _require(a.dtype == np.int32 and a.flags["C_CONTIGUOUS"], "expected a C-contiguous int32 array")
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _ptr_array(ptrs: Sequence[int]):
    arr = (ctypes.POINTER(ctypes.c_int32) * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = ctypes.cast(ctypes.c_void_p(p), ctypes.POINTER(ctypes.c_int32))
    return arr


@dataclass
class WarpBatchInput:
    """A batch of ``WarpInput`` (interp.hpp:14-22) in the compact layout."""

    kernel: str
    warp: int
    n_warps: int
    args: np.ndarray                      # (n_params, acount) int32
    globals: Dict[str, np.ndarray]        # name -> (n_warps*gstride,) int32
    shared: Dict[str, np.ndarray] = field(default_factory=dict)  # name -> (n_warps*size,)
    gstride: int = 0
    seed0: int = 0


def make_random_input(kernel: str, warp: int, n_warps: int, seed0: int,
                      gstride: Optional[int] = None) -> WarpBatchInput:
    """``makeRandomInput(m, f, warp, seed0 + w)`` for w in [0, n_warps).

    ``gstride`` words of every global are kept per warp (default: ``warp``, the
    words the corpus kernels can touch); pass the declared size to keep all.
    """
    info = kernel_info(kernel)
    gstride = warp if gstride is None else gstride
    np_ = len(info["params"])
    args = np.zeros((max(np_, 1), n_warps), dtype=np.int32)
    gl = {name: np.zeros(n_warps * gstride, dtype=np.int32) for name, _ in info["globals"]}
    sh = {name: np.zeros(n_warps * size, dtype=np.int32) for name, size in info["shared"]}
    err = ctypes.create_string_buffer(512)
    rc = lib().darm_gpu_make_random_input(
        kernel.encode(), warp, n_warps, seed0, _i32p(args),
        _ptr_array([gl[n].ctypes.data for n, _ in info["globals"]]), gstride,
        _ptr_array([sh[n].ctypes.data for n, _ in info["shared"]]) if sh else None, err, 512)
    _check(rc, err)
    return WarpBatchInput(kernel, warp, n_warps, args[:np_], gl, sh, gstride, seed0)


@dataclass
class WarpBatchResult:
    """``WarpResult`` (interp.hpp:41-53) for a batch: final globals + fault counts."""

    globals: Dict[str, np.ndarray]
    faults: np.ndarray
    stats: dict


def _require(ok, what):
    """Argument check of the public wrappers: a DarmUserError (the C-ABI's
    user-error class, code 2), not an assert, so it holds under python -O."""
    if not ok:
        raise DarmUserError(what)


def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _require_i32(x, name, min_words=0):
    """A DEVICE (torch CUDA) or HOST (numpy) int32 buffer the C-ABI may walk
    as ``min_words`` contiguous words."""
    if _is_torch_cuda(x):
        import torch

        _require(x.dtype == torch.int32 and x.is_contiguous(), f"{name}: expected a contiguous int32 CUDA tensor")
        _require(x.numel() >= min_words, f"{name}: {x.numel()} words, at least {min_words} needed")
    else:
        _require(isinstance(x, np.ndarray) and x.dtype == np.int32 and x.flags["C_CONTIGUOUS"],
                 f"{name}: expected a C-contiguous int32 numpy array or int32 CUDA tensor")
        _require(x.size >= min_words, f"{name}: {x.size} words, at least {min_words} needed")


def execute_warps(kernel: str, variant, warp: int, args, globals: Dict[str, object],
                  shared: Optional[Dict[str, object]] = None, n_warps: Optional[int] = None,
                  faults=None, stream=None, want_stats: bool = True, prepare_only: bool = False,
                  count_faults: bool = True):
    """Run a batch of warps of a corpus kernel on the GPU (replaces executeWarp).

    ``globals``/``shared`` are numpy int32 arrays (HOST mode: copied in and the
    globals copied back in place) or torch int32 CUDA tensors (DEVICE mode:
    updated in place, asynchronous on ``stream``).  ``args`` is an int32 array of
    shape (n_params, acount) with acount in {1, n_warps, n_warps*warp}; with
    acount == 1 it is always host memory.  ``prepare_only`` returns a
    :class:`PreparedCall` instead of running.  ``count_faults=False`` passes
    no fault counters (kernels without shared memory then launch one kernel
    and nothing else; their lanes are in bounds by construction).
    """
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    info = kernel_info(kernel)
    names = [n for n, _ in info["globals"]]
    snames = [n for n, _ in info["shared"]]
    first = globals[names[0]]
    device = _is_torch_cuda(first)
    n_lanes = int(first.numel() if device else first.size)
    if n_warps is None:
        n_warps = n_lanes // warp
    for n in names:   # compact batch layout: word w*warp + t of every global
        _require(n in globals, f"missing global {n}")
        _require(_is_torch_cuda(globals[n]) == device, f"{n}: globals must all be numpy or all CUDA tensors")
        _require_i32(globals[n], n, n_warps * warp)
    for n, size in info["shared"]:
        if shared:
            _require(n in shared, f"missing shared {n}")
            _require(_is_torch_cuda(shared[n]) == device, f"{n}: shared must be the same memory kind as globals")
            _require_i32(shared[n], n, n_warps * size)
    if faults is not None:
        _require_i32(faults, "faults", n_warps)
    if device:
        import torch

        args_t = args if _is_torch_cuda(args) else None
        if args_t is None:
            args_np = np.ascontiguousarray(np.asarray(args, dtype=np.int32).reshape(len(info["params"]), -1))
            acount = args_np.shape[1]
            if acount != 1:
                args_t = torch.from_numpy(args_np).to(first.device)
        else:
            acount = args_t.shape[-1]
        if acount == 1 and args_t is None:
            aptr = _i32p(args_np)
        else:
            aptr = ctypes.cast(ctypes.c_void_p(args_t.data_ptr()), ctypes.POINTER(ctypes.c_int32))
        gl_ptrs = [globals[n].data_ptr() for n in names]
        sh_ptrs = [shared[n].data_ptr() for n in snames] if shared else []
        if faults is None and count_faults:
            faults = torch.zeros(n_warps, dtype=torch.int32, device=first.device)
        fptr = (ctypes.cast(ctypes.c_void_p(faults.data_ptr()), ctypes.POINTER(ctypes.c_int32))
                if faults is not None else None)
        mem = 1
        if stream is None:
            stream = torch.cuda.current_stream(first.device).cuda_stream
        elif args_t is not None and args_t is not args:
            # allocated on the current stream, read on `stream`: keep the
            # caching allocator from reusing it before the launch has run
            args_t.record_stream(torch.cuda.ExternalStream(int(stream), device=first.device))
    else:
        args_np = np.ascontiguousarray(np.asarray(args, dtype=np.int32).reshape(len(info["params"]), -1))
        acount = args_np.shape[1]
        aptr = _i32p(args_np)
        gl_ptrs = [globals[n].ctypes.data for n in names]
        sh_ptrs = [shared[n].ctypes.data for n in snames] if shared else []   # checked int32, C-contiguous
        if faults is None:
            faults = np.zeros(n_warps, dtype=np.int32)
        fptr = _i32p(faults)
        mem = 0
    call = PreparedCall(lib().darm_gpu_execute_warps, (
        kernel.encode(), int(variant), int(warp), int(n_warps), aptr, int(acount),
        _ptr_array(gl_ptrs), len(gl_ptrs), _ptr_array(sh_ptrs) if sh_ptrs else None, len(sh_ptrs),
        fptr, mem, ctypes.c_void_p(stream or 0)), want_stats,
        keepalive=(args_np if not device or acount == 1 else args_t, globals, shared, faults))
    if prepare_only:
        return call
    st = call()
    return WarpBatchResult({n: globals[n] for n in names}, faults, st)


class PreparedCall:
    """One C-ABI call with its ctypes arguments built once; calling it costs a
    single foreign call (used by bench.py so host overhead stays off the GPU
    timeline).  Holds references to every buffer the pointers refer to."""

    def __init__(self, fn, args, want_stats, keepalive=()):
        self.fn, self.args, self.keepalive = fn, args, keepalive
        self.stats = Stats() if want_stats else None
        self.err = ctypes.create_string_buffer(512)
        self.full = args + ((ctypes.byref(self.stats) if want_stats else None), self.err, 512)

    def __call__(self) -> dict:
        _check(self.fn(*self.full), self.err)
        return self.stats.as_dict() if self.stats is not None else {}


def _network_sort(fn, keys, bucket, variant, stream, want_stats, prepare_only, keys_per_thread):
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    _require_i32(keys, "keys")
    if _is_torch_cuda(keys):
        import torch

        ptr, n, mem = keys.data_ptr(), keys.numel(), 1
        if stream is None:
            stream = torch.cuda.current_stream(keys.device).cuda_stream
    else:
        ptr, n, mem = keys.ctypes.data, keys.size, 0
    call = PreparedCall(fn, (int(variant), ctypes.c_void_p(ptr), int(n), int(bucket), int(keys_per_thread), mem,
                             ctypes.c_void_p(stream or 0)), want_stats, keepalive=(keys,))
    return call if prepare_only else call()


def bitonic_sort(keys, bucket: int, variant=MELDED, stream=None, want_stats: bool = True,
                 prepare_only: bool = False, keys_per_thread: int = 0):
    """Sort every ``bucket``-key bucket of ``keys`` ascending, in place, by the
    chain of corpus bitonic.ir steps.

    ``keys``: numpy int32 (HOST mode) or torch int32 CUDA tensor (DEVICE mode).
    ``keys_per_thread``: 1 = one key per thread (the IR warp shape), 4/8/16 =
    register-blocked, 0 = fastest (``darm_gpu_bitonic_sort_ex``).  The stats
    dict reports the choice as ``keys_per_thread``.
    """
    return _network_sort(lib().darm_gpu_bitonic_sort_ex, keys, bucket, variant, stream, want_stats, prepare_only,
                         keys_per_thread)


def oddeven_sort(keys, bucket: int, variant=MELDED, stream=None, want_stats: bool = True,
                 prepare_only: bool = False, keys_per_thread: int = 0):
    """PCM: Batcher odd-even merge sort of every ``bucket``-key bucket, in place,
    by the chain of ir/oddeven_step.ir steps (``darm_gpu_oddeven_sort``);
    arguments as :func:`bitonic_sort`."""
    return _network_sort(lib().darm_gpu_oddeven_sort, keys, bucket, variant, stream, want_stats, prepare_only,
                         keys_per_thread)


def merge_sort(keys, variant=MELDED, stream=None, want_stats: bool = True, prepare_only: bool = False):
    """MS: bottom-up merge sort of the whole of ``keys`` (int32, numpy HOST or
    torch CUDA), in place, by the merge loop of ir/merge_step.ir
    (``darm_gpu_merge_sort``)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    _require_i32(keys, "keys")
    if _is_torch_cuda(keys):
        import torch

        ptr, n, mem = keys.data_ptr(), keys.numel(), 1
        if stream is None:
            stream = torch.cuda.current_stream(keys.device).cuda_stream
    else:
        ptr, n, mem = keys.ctypes.data, keys.size, 0
    call = PreparedCall(lib().darm_gpu_merge_sort, (int(variant), ctypes.c_void_p(ptr), int(n), mem,
                                                    ctypes.c_void_p(stream or 0)), want_stats, keepalive=(keys,))
    return call if prepare_only else call()


@dataclass
class ProgramResult:
    """WarpResult fields for a batch (interp.hpp:41-53): ``returns`` /
    ``ret_valid`` [n_warps, warp], ``globals`` / ``shared`` [n_warps, words]
    (final memories), ``faults`` [n_warps], ``stats`` [n_warps, 8] in the
    order issuedInstructions, threadCycles, usefulThreadCycles,
    serializedCycles, divergentBranchCount, sharedMemIssues, globalMemIssues,
    flags (bit 0 nonTerminated, bit 1 taintedObservable)."""
    returns: object
    ret_valid: object
    globals: object
    shared: object
    faults: object
    stats: object
    call_stats: dict = field(default_factory=dict)

    @property
    def utilization(self):
        thread, useful = self.stats[:, 1], self.stats[:, 2]
        return np.where(thread == 0, 1.0, useful / np.maximum(thread, 1))


class Program:
    """A mini-IR function (the reference's textual IR) loaded
    into the GPU warp interpreter: :meth:`execute_warps` is executeWarp
    (interp.hpp:57-58) for a batch of warps of ANY function, results equal to
    the reference interpreter's (``darm_gpu_program_*``)."""

    def __init__(self, ir_text: str, latency: Optional[Sequence[int]] = None):
        err = ctypes.create_string_buffer(512)
        h = ctypes.c_void_p()
        lat = None
        if latency is not None:
            lat = (ctypes.c_int64 * 28)(*[int(x) for x in latency])
        _check(lib().darm_gpu_program_load(ir_text.encode(), lat, ctypes.byref(h), err, 512), err)
        self.h = h
        np_, ng, ns = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        gw, sw = ctypes.c_int64(), ctypes.c_int64()
        lib().darm_gpu_program_shape(h, ctypes.byref(np_), ctypes.byref(ng), ctypes.byref(ns), ctypes.byref(gw),
                                     ctypes.byref(sw))
        self.params = [lib().darm_gpu_program_param(h, i).decode() for i in range(np_.value)]
        self.memories = []   # (name, size, offset, is_shared) — globals, then shared arrays
        for i in range(ng.value + ns.value):
            size, off, sh = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
            name = lib().darm_gpu_program_memory(h, i, ctypes.byref(size), ctypes.byref(off), ctypes.byref(sh))
            self.memories.append((name.decode(), size.value, off.value, bool(sh.value)))
        self.global_words, self.shared_words = gw.value, sw.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().darm_gpu_program_free(self.h)
                self.h = None
        except Exception:
            pass

    def execute_warps(self, warp: int, args, globals_, shared=None, max_steps: int = 0, stream=None,
                      want_stats: bool = True, n_warps: Optional[int] = None) -> ProgramResult:
        """``args``: [n_params, acount] (acount 1, n_warps or n_warps*warp);
        ``globals_``: [n_warps, global_words] int32, updated in place;
        ``shared``: [n_warps, shared_words] or None (zeros); ``n_warps``
        defaults to ``globals_.shape[0]``.  numpy arrays run through HOST
        buffers, torch CUDA tensors in place (DEVICE)."""
        dev = _is_torch_cuda(globals_)
        if n_warps is None:
            n_warps = int(globals_.shape[0])
        _require_i32(globals_, "globals", n_warps * self.global_words)
        if shared is not None:
            _require(_is_torch_cuda(shared) == dev, "shared: same memory kind as globals")
            _require_i32(shared, "shared", n_warps * self.shared_words)
        if dev:
            import torch

            ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
            args_t = torch.as_tensor(np.asarray(args, np.int32) if not _is_torch_cuda(args) else args,
                                     device=globals_.device).to(torch.int32).contiguous()
            rets = torch.zeros((n_warps, warp), dtype=torch.int32, device=globals_.device)
            valid = torch.zeros((n_warps, warp), dtype=torch.uint8, device=globals_.device)
            faults = torch.zeros(n_warps, dtype=torch.int32, device=globals_.device)
            stats = torch.zeros((n_warps, 8), dtype=torch.int64, device=globals_.device)
            if stream is None:
                stream = torch.cuda.current_stream(globals_.device).cuda_stream
            mem, keep = 1, (args_t,)
            a_ptr = ptr(args_t)
            acount = args_t.shape[-1] if args_t.numel() else 1
        else:
            args_n = np.ascontiguousarray(args, dtype=np.int32)
            rets = np.zeros((n_warps, warp), np.int32)
            valid = np.zeros((n_warps, warp), np.uint8)
            faults = np.zeros(n_warps, np.int32)
            stats = np.zeros((n_warps, 8), np.int64)
            ptr = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else None  # noqa: E731
            mem, keep = 0, (args_n,)
            a_ptr = ptr(args_n) if args_n.size else None
            acount = args_n.shape[-1] if args_n.size else 1
        st = Stats()
        err = ctypes.create_string_buffer(512)
        rc = lib().darm_gpu_program_execute(self.h, warp, n_warps, a_ptr, acount, ptr(globals_), ptr(shared),
                                            ptr(rets), ptr(valid), ptr(faults), ptr(stats), int(max_steps), mem,
                                            ctypes.c_void_p(stream or 0), ctypes.byref(st) if want_stats else None,
                                            err, 512)
        del keep
        _check(rc, err)
        return ProgramResult(rets, valid, globals_, shared, faults, stats, st.as_dict() if want_stats else {})


NQ_MIRROR, NQ_PAPER_SHAPE = 1, 2     # darm_gpu.h DARM_NQ_*


def nqueens(n: int, prefix_rows: int, variant=MELDED, rank: int = 0, world: int = 1,
            per_prefix: bool = False, stream=None, want_stats: bool = True, mirror: bool = False,
            paper_shape: bool = False):
    """Count n-queens solutions below the prefixes i % world == rank.

    ``mirror``: count by mirror symmetry (half the search, DARM_NQ_MIRROR).
    ``paper_shape``: run ir/nqueens_step.ir (pop / leaf / push, the paper's
    if-then-elseif-then melded by region replication) instead of the
    symmetric encoding (DARM_NQ_PAPER_SHAPE, n <= 16).
    Returns ``(solutions, per_prefix_counts or None, stats)``.
    """
    flags = (NQ_MIRROR if mirror else 0) | (NQ_PAPER_SHAPE if paper_shape else 0)
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    sols = ctypes.c_uint64(0)
    npre = ctypes.c_int64(0)
    err = ctypes.create_string_buffer(512)
    per = None
    if per_prefix:
        cnt = lib().darm_gpu_nqueens_prefix_count_ex(n, prefix_rows, rank, world, flags & NQ_MIRROR)
        if cnt < 0:
            raise DarmUserError("bad n-queens arguments")
        per = np.zeros(max(1, cnt), dtype=np.uint32)
    st = Stats()
    rc = lib().darm_gpu_nqueens_ex(
        int(variant), n, prefix_rows, rank, world, flags, ctypes.byref(sols),
        per.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)) if per is not None else None,
        per.size if per is not None else 0, ctypes.byref(npre), ctypes.c_void_p(stream or 0),
        ctypes.byref(st) if want_stats else None, err, 512)
    _check(rc, err)
    return int(sols.value), (per[: npre.value] if per is not None else None), (st.as_dict() if want_stats else {})


def lud(a, variant=MELDED, stream=None, want_stats: bool = True, prepare_only: bool = False):
    """In-place blocked LU (no pivoting) of a square fp32 matrix.

    ``a``: numpy float32 (HOST mode) or torch float32 CUDA tensor (DEVICE mode),
    row-major n x n with n % 16 == 0.
    """
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    if _is_torch_cuda(a):
        import torch

        _require(a.dtype == torch.float32 and a.is_contiguous() and a.dim() == 2 and a.shape[0] == a.shape[1],
                 "a: expected a contiguous square float32 CUDA tensor")
        ptr, n, mem = a.data_ptr(), a.shape[0], 1
        if stream is None:
            stream = torch.cuda.current_stream(a.device).cuda_stream
    else:
        _require(a.dtype == np.float32 and a.flags["C_CONTIGUOUS"] and a.ndim == 2 and a.shape[0] == a.shape[1],
                 "a: expected a C-contiguous square float32 array")
        ptr, n, mem = a.ctypes.data, a.shape[0], 0
    call = PreparedCall(lib().darm_gpu_lud, (int(variant), ctypes.c_void_p(ptr), int(n), mem,
                                             ctypes.c_void_p(stream or 0)), want_stats, keepalive=(a,))
    return call if prepare_only else call()


RODINIA_ROI = (0, 127, 0, 127)


def _roi_arr(roi):
    r = (ctypes.c_int32 * 4)(*[int(x) for x in roi])
    return r


def srad(j, iters: int, lam: float = 0.5, roi=RODINIA_ROI, variant=MELDED, stream=None,
         want_stats: bool = True, prepare_only: bool = False, fast: bool = False):
    """SRAD on a 2-D fp32 image, in place (numpy -> HOST mode, torch CUDA -> DEVICE).
    ``fast``: reciprocal-multiply divisions and FMAs (DARM_FAST_MATH; within
    1e-5 relative of the IEEE path instead of bit-identical)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    if fast:
        variant |= FAST_MATH
    if _is_torch_cuda(j):
        import torch

        _require(j.dtype == torch.float32 and j.is_contiguous() and j.dim() == 2,
                 "j: expected a contiguous 2-D float32 CUDA tensor")
        ptr, (rows, cols), mem = j.data_ptr(), j.shape, 1
        if stream is None:
            stream = torch.cuda.current_stream(j.device).cuda_stream
    else:
        _require(j.dtype == np.float32 and j.flags["C_CONTIGUOUS"] and j.ndim == 2,
                 "j: expected a C-contiguous 2-D float32 array")
        ptr, (rows, cols), mem = j.ctypes.data, j.shape, 0
    r = _roi_arr(roi)
    call = PreparedCall(lib().darm_gpu_srad, (int(variant), ctypes.c_void_p(ptr), int(rows), int(cols), int(iters),
                                              float(lam), r, mem, ctypes.c_void_p(stream or 0)), want_stats,
                        keepalive=(j, r))
    return call if prepare_only else call()


def srad_roi_words(cols: int, roi=RODINIA_ROI) -> int:
    return int(lib().darm_gpu_srad_roi_words(int(cols), _roi_arr(roi)))


def srad_pitch(cols: int) -> int:
    """Row pitch (floats) of SRAD tile buffers: cols rounded up to a multiple of 4."""
    return (int(cols) + 3) & ~3


def srad_tile_roi(tile, cols, tile_rows, r0, rows, roi, roi_out, stream=None) -> None:
    """ROI partials of a tile (device tensors, rows of tile.shape[1] floats; see darm_gpu.h)."""
    err = ctypes.create_string_buffer(512)
    _check(lib().darm_gpu_srad_tile_roi(ctypes.c_void_p(tile.data_ptr()), cols, tile.shape[1], tile_rows, r0, rows,
                                        _roi_arr(roi), ctypes.c_void_p(roi_out.data_ptr()),
                                        ctypes.c_void_p(stream or 0), err, 512), err)


def srad_tile_step(variant, tile_in, tile_out, cols, tile_rows, r0, rows, lam, roi, roi_in, roi_out, q0,
                   stream=None, part: int = SRAD_ALL_ROWS) -> None:
    """One SRAD iteration of a row tile, or its interior / edge rows (`part`;
    device tensors, rows of tile_in.shape[1] floats; see darm_gpu.h)."""
    if isinstance(variant, str):
        variant = VARIANTS[variant]
    _require(tile_in.shape == tile_out.shape, "tile_in and tile_out must have the same shape")
    err = ctypes.create_string_buffer(512)
    _check(lib().darm_gpu_srad_tile_step(int(variant), ctypes.c_void_p(tile_in.data_ptr()),
                                         ctypes.c_void_p(tile_out.data_ptr()), cols, tile_in.shape[1], tile_rows, r0,
                                         rows, float(lam), _roi_arr(roi), ctypes.c_void_p(roi_in.data_ptr()),
                                         ctypes.c_void_p(roi_out.data_ptr()), ctypes.c_void_p(q0.data_ptr()),
                                         int(part), ctypes.c_void_p(stream or 0), err, 512), err)


@dataclass
class CompareVerdict:
    equal: bool = True
    diff: str = ""
    warp: int = -1


def compare_runs(a: WarpBatchResult, b: WarpBatchResult, warp: int, gstride: Optional[int] = None) -> CompareVerdict:
    """``compareRuns`` (interp.cpp:383-426) slice by slice: fault counts, then
    global memories (shared memory is not compared).  Corpus kernels return
    void, so the per-lane return comparison is vacuous."""
    def host(x):
        return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)

    fa, fb = host(a.faults), host(b.faults)
    bad = np.nonzero(fa != fb)[0]
    first_fault = int(bad[0]) if bad.size else None
    first_mem, mem_name = None, ""
    for name in a.globals:
        ga, gb = host(a.globals[name]), host(b.globals[name])
        stride = gstride or warp
        diff = np.nonzero((ga != gb).reshape(-1, stride).any(axis=1))[0]
        if diff.size and (first_mem is None or diff[0] < first_mem):
            first_mem, mem_name = int(diff[0]), name
    cands = [w for w in (first_fault, first_mem) if w is not None]
    if not cands:
        return CompareVerdict()
    w = min(cands)
    if first_fault is not None and first_fault == w:
        return CompareVerdict(False, "fault counts differ", w)
    return CompareVerdict(False, f"global memory '{mem_name}' differs", w)


def shutdown() -> None:
    """Release the library's cached device buffers."""
    if _lib is not None:
        _lib.darm_gpu_shutdown()
