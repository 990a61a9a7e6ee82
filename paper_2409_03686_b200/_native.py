"""ctypes binding of libexitmeasure_b200.so (include/exitmeasure_b200.h).

This replaces the reference's Cython binding of its kernel
(S/_kernel.pyx:376-464, S/ = /root/reference/pkg/src/exitmeasure/).  There is
no CPU fallback: if the library is missing or no CUDA device is visible, the
first call raises ``NativeError``.  ctypes releases the GIL for the duration
of every foreign call, which keeps the reference's thread-pool contract
(S/_kernel.pyx:398,435) for callers that still drive chunks from threads.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import NativeError

# EXITMEASURE_B200_DEBUG=1 loads the EM_DEBUG variant (device bounds asserts)
DEBUG = os.environ.get("EXITMEASURE_B200_DEBUG") == "1"
LIB_PATH = (Path(__file__).resolve().parent / "lib"
            / ("libexitmeasure_b200_debug.so" if DEBUG else "libexitmeasure_b200.so"))
# A/B tooling only (tools/diag/x2_variants.sh): load a variant build instead;
# em_build_info() in every bench line says what was loaded
if os.environ.get("EXITMEASURE_B200_LIB"):
    LIB_PATH = Path(os.environ["EXITMEASURE_B200_LIB"]).resolve()

EM_OK = 0
EM_BUDGET = 1
EM_ERR_INVALID = -1
EM_ERR_CUDA = -2
EM_ERR_UNSUPPORTED = -3
EM_ERR_NOMEM = -4
EM_PREC_REF64 = 0
EM_PREC_FP32 = 1
EM_CHAIN_WOE = 0
EM_CHAIN_MAX = 1
EM_CHAIN_TANGENT = 2
EM_FLAG_TANGENT_ON_IDENTITY = 1
EM_FLAG_PERSISTENT = 2
EM_FLAG_POLE_BLOCKS = 4
EM_FLAG_ONE_WALK_PER_LANE = 8
EM_FLAG_TWO_WALKS_PER_LANE = 16

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_p = ctypes.c_void_p
_dbl = ctypes.c_double


class EmGeometry(ctypes.Structure):
    _fields_ = [("gi", _p), ("gi_len", _i64), ("gf", _p), ("gf_len", _i64),
                ("comp_side", _p), ("n_comp", _i64), ("ksqrt", _p)]


class EmSide(ctypes.Structure):
    _fields_ = [("anchors", _p), ("n_anchors", _i64), ("blk", _p), ("blkf", _p),
                ("n_blk", _i64), ("wkind", _i32), ("idw_power", _i32),
                ("idw_radii", _p), ("blk_phase", _p)]


class EmOptions(ctypes.Structure):
    _fields_ = [("precision", _i32), ("chain", _i32), ("device", _i32), ("block", _i32),
                ("grid", _i32), ("flags", _i32)]


class EmOutputs(ctypes.Structure):
    _fields_ = [("counts", _p), ("steps_sum", _p), ("steps_sq", _p), ("steps_max", _p),
                ("err_pole", _i64), ("err_rep", _i64)]


_lib = None


def lib():
    """Load the CUDA library (built in-tree by build_native.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if os.environ.get("EXITMEASURE_B200_AUTOBUILD", "1") == "1":
            from .build_native import build

            build(debug=DEBUG)
        if not LIB_PATH.exists():
            raise NativeError(f"CUDA library missing: {LIB_PATH} "
                              "(run python -m paper_2409_03686_b200.build_native)")
    L = ctypes.CDLL(str(LIB_PATH))
    sig = {
        "em_abi_version": ([], ctypes.c_int),
        "em_build_info": ([], ctypes.c_char_p),
        "em_last_error": ([], ctypes.c_char_p),
        "em_device_count": ([], ctypes.c_int),
        "em_device_info": ([ctypes.c_int, _p, _p, _p, _p], ctypes.c_int),
        "em_walk_exits_chunk": ([ctypes.POINTER(EmGeometry), _p, _i64, _i64, _i64, _u64, _dbl,
                                 _i64, ctypes.c_int, _p, _p, _p, _p], ctypes.c_int),
        "em_accumulate_chunk": ([ctypes.POINTER(EmGeometry), _p, _i64, _i64, _i64, _u64, _dbl,
                                 _i64, ctypes.POINTER(EmSide), ctypes.POINTER(EmSide),
                                 ctypes.c_int, _p, _p, _p, _p], ctypes.c_int),
        "em_plan_create": ([ctypes.POINTER(EmGeometry), ctypes.POINTER(EmSide),
                            ctypes.POINTER(EmSide), _p, _p, _i64, _dbl, _i64,
                            ctypes.POINTER(EmOptions), ctypes.POINTER(_p)], ctypes.c_int),
        "em_plan_destroy": ([_p], ctypes.c_int),
        "em_plan_run": ([_p, _u64, _i64, _i64, ctypes.POINTER(EmOutputs)], ctypes.c_int),
        "em_plan_run_host": ([_p, _u64, _i64, _i64, ctypes.POINTER(ctypes.POINTER(_i64)), _p, _p],
                             ctypes.c_int),
        "em_plan_run_host_f64": ([_p, _u64, _i64, _i64, ctypes.POINTER(ctypes.POINTER(_i64)),
                                  _p, _p], ctypes.c_int),
        "em_plan_detach_block": ([_p, ctypes.POINTER(ctypes.POINTER(_i64))], ctypes.c_int),
        "em_host_block_free": ([_p], ctypes.c_int),
        "em_plan_run_device": ([_p, _u64, _i64, _i64, ctypes.POINTER(EmOutputs), _p],
                               ctypes.c_int),
        "em_plan_last_stats": ([_p, _p, _p, _p], ctypes.c_int),
        "em_plan_check": ([_p, _p, _p], ctypes.c_int),
        "em_plan_last_launches": ([_p, _p], ctypes.c_int),
        "em_plan_chain": ([_p], ctypes.c_int),
        "em_resolve_chain": ([ctypes.POINTER(EmGeometry), ctypes.c_int, ctypes.c_int],
                             ctypes.c_int),
        "em_plan_n_bins": ([_p, ctypes.c_int], _i64),
        "em_plan_last_scheduler": ([_p], ctypes.c_int),
        "em_plan_walks_per_lane": ([_p], ctypes.c_int),
        "em_plan_last_walks_per_lane": ([_p], ctypes.c_int),
        "em_run_accumulate": ([ctypes.POINTER(EmGeometry), ctypes.POINTER(EmSide),
                               ctypes.POINTER(EmSide), _p, _p, _i64, _u64, _dbl, _i64, _i64,
                               ctypes.POINTER(EmOptions), ctypes.POINTER(EmOutputs)],
                              ctypes.c_int),
        "em_run_exits": ([_p, _u64, _i64, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
        "em_plan_run_raw": ([_p, _u64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p],
                            ctypes.c_int),
        "em_bin_points": ([_p, _p, _i64, _p, _p, _p], ctypes.c_int),
        "em_debug_step": ([_p, _p, _p, _i64, _p, _p], ctypes.c_int),
        "em_f32_constant": ([ctypes.POINTER(EmGeometry), ctypes.c_int, ctypes.c_int, _dbl,
                             ctypes.c_char_p, _p, ctypes.c_int], ctypes.c_int),
        "em_fp32_peak": ([ctypes.c_int, _p, _p], ctypes.c_int),
        "em_philox4x64_blocks": ([_p, _p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "em_philox4x32_blocks": ([_p, _p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "em_curand_philox4x32_blocks": ([_p, _p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.em_abi_version() != 1:
        raise NativeError("libexitmeasure_b200 ABI mismatch")
    _lib = L
    return L


def declared_symbols() -> list:
    """Function names declared in include/exitmeasure_b200.h."""
    import re

    text = (Path(__file__).resolve().parents[1] / "include" / "exitmeasure_b200.h").read_text()
    return re.findall(r"^(?:int|const char\*|int64_t)\s+\*?(em_\w+)\s*\(", text, re.M)


def exported_symbols():
    """(name, exported?) for every function the header declares."""
    L = ctypes.CDLL(str(LIB_PATH))
    return [(n, hasattr(L, n)) for n in declared_symbols()]


def build_info() -> dict:
    """The compile knobs of the loaded library (em_build_info) as a dict."""
    text = lib().em_build_info().decode()
    return dict(kv.split("=", 1) for kv in text.split())


def last_error() -> str:
    return lib().em_last_error().decode(errors="replace")


def check(rc: int, what: str) -> int:
    """Raise NativeError on negative return codes; pass EM_OK / EM_BUDGET."""
    if rc < 0:
        raise NativeError(f"{what} failed ({rc}): {last_error()}")
    return rc


def device_count() -> int:
    return int(lib().em_device_count())


_seen_devices = 0


def require_device(device: int = 0) -> None:
    global _seen_devices
    if device < _seen_devices:  # visible devices do not go away within a process
        return
    n = device_count()
    _seen_devices = n
    if device >= n:
        raise NativeError(f"no CUDA device {device} ({n} visible): the exit-measure "
                          "path runs on the GPU only (no CPU fallback)")


def device_info(device: int = 0) -> dict:
    v = [ctypes.c_int(0) for _ in range(4)]
    check(lib().em_device_info(device, *[ctypes.byref(x) for x in v]), "em_device_info")
    return {"sm_count": v[0].value, "clock_khz": v[1].value, "cc": (v[2].value, v[3].value)}


def ptr(a: np.ndarray):
    # the raw address as a Python int (c_void_p arguments and struct fields
    # accept it); a.ctypes.data_as costs ~5 us per call on the API path
    return a.__array_interface__["data"][0]


def fp32_peak(device: int = 0):
    f = ctypes.c_double(0)
    ms = ctypes.c_double(0)
    check(lib().em_fp32_peak(device, ctypes.byref(f), ctypes.byref(ms)), "em_fp32_peak")
    return f.value, ms.value


def philox4x64_blocks(inputs: np.ndarray, device: int = 0) -> np.ndarray:
    """inputs (n, 6) uint64 = (c0, c1, c2, c3, k0, k1) -> (n, 4) uint64."""
    a = np.ascontiguousarray(inputs, dtype=np.uint64)
    out = np.zeros((a.shape[0], 4), dtype=np.uint64)
    check(lib().em_philox4x64_blocks(ptr(a), ptr(out), a.shape[0], device), "philox64")
    return out


def philox4x32_blocks(inputs: np.ndarray, device: int = 0, curand: bool = False) -> np.ndarray:
    """inputs (n, 6) uint32 = (c0, c1, c2, c3, k0, k1) -> (n, 4) uint32;
    curand=True evaluates the toolkit's curand_Philox4x32_10 instead."""
    a = np.ascontiguousarray(inputs, dtype=np.uint32)
    out = np.zeros((a.shape[0], 4), dtype=np.uint32)
    f = lib().em_curand_philox4x32_blocks if curand else lib().em_philox4x32_blocks
    check(f(ptr(a), ptr(out), a.shape[0], device), "philox32")
    return out
