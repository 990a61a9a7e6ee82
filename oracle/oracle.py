"""ctypes front end of the CPU parity oracle (``oracle/em_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline legs, always as the checker or the timed CPU
baseline, never by the product package (``paper_2409_03686_b200``).

The module exposes the reference's ``_impl`` chunk contract
(``walk_exits_chunk`` / ``accumulate_chunk``, S/_kernel.pyx:376-464 with
S/ = /root/reference/pkg/src/exitmeasure/) and the driver
``run_accumulate`` (S/backend.py:147-199), with identical argument meaning, so
a test can swap it in wherever the reference's compiled kernel is used.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libem_oracle.so"

_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_p = ctypes.c_void_p


class EmoSide(ctypes.Structure):
    """Mirror of ``emo_side`` (em_oracle.h); one packed weight family."""

    _fields_ = [
        ("anchors", _p), ("n_anchors", _i64), ("blk", _p), ("blkf", _p),
        ("n_blk", _i64), ("wkind", ctypes.c_int32), ("idw_power", ctypes.c_int32),
        ("idw_radii", _p),
    ]


def build() -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.emo_philox4x64.argtypes = [_u64] * 6 + [_p]
        L.emo_philox4x64.restype = None
        L.emo_signed_dist.argtypes = [_p, _i64, _p, _p]
        L.emo_signed_dist.restype = _dbl
        L.emo_owner_component.argtypes = [_p, _i64, _p, _p]
        L.emo_owner_component.restype = _i64
        L.emo_assign_anchor.argtypes = [_p, ctypes.c_int, ctypes.POINTER(EmoSide)]
        L.emo_assign_anchor.restype = _i64
        L.emo_walk_exits_chunk.argtypes = [_p, _i64, _p, _p, _p, _i64, _i64, _i64,
                                           _u64, _dbl, _i64, _p, _p, _p]
        L.emo_walk_exits_chunk.restype = _i64
        L.emo_accumulate_chunk.argtypes = [_p, _i64, _p, _p, _p, _p, _i64, _i64, _i64,
                                           _u64, _dbl, _i64, ctypes.POINTER(EmoSide),
                                           ctypes.POINTER(EmoSide), _p, _p, _p]
        L.emo_accumulate_chunk.restype = _i64
        L.emo_run_accumulate.argtypes = [_p, _i64, _p, _p, _p, _p, _i64, _u64, _dbl,
                                         _i64, _i64, ctypes.POINTER(EmoSide),
                                         ctypes.POINTER(EmoSide), _p, _p, _p, _p, _p,
                                         _p, _p, ctypes.c_int]
        L.emo_run_accumulate.restype = _i64
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def philox4x64(key0, c0, c1, c2, c3, key1=0):
    """One Philox4x64-10 block (S/_kernel.pyx:37-54) -> 4 Python ints."""
    out = np.zeros(4, dtype=np.uint64)
    lib().emo_philox4x64(int(key0), int(key1), int(c0), int(c1), int(c2), int(c3),
                         _ptr(out))
    return [int(w) for w in out]


def _side(anchors, blk, blkf, wkind=0, idw_radii=None, idw_power=2, keep=None):
    anchors = _c(anchors, np.float64)
    blk = _c(blk, np.int64).reshape(-1, 3)
    blkf = _c(blkf, np.float64).reshape(-1, 4)
    radii = _c(idw_radii if idw_radii is not None else np.zeros(0), np.float64)
    if keep is not None:
        keep.extend([anchors, blk, blkf, radii])
    return EmoSide(_ptr(anchors), anchors.shape[0], _ptr(blk), _ptr(blkf),
                   blk.shape[0], int(wkind), int(idw_power), _ptr(radii))


def walk_exits_chunk(gi, gf, comp_side, ksqrt, pole_xy, pole_index, rep_start,
                     rep_end, seed, eps, max_steps):
    """Same contract as the reference's _kernel.walk_exits_chunk."""
    gi = _c(gi, np.int64)
    gf = _c(gf, np.float64)
    ks = _c(ksqrt, np.float64)
    pole = _c(pole_xy, np.float64)
    d = int(gi[0])
    n = int(rep_end) - int(rep_start)
    x = np.empty((n, d))
    steps = np.empty(n, dtype=np.int64)
    comp = np.empty(n, dtype=np.int64)
    err = lib().emo_walk_exits_chunk(_ptr(gi), gi.shape[0], _ptr(gf), _ptr(ks), _ptr(pole),
                                     int(pole_index), int(rep_start), int(rep_end),
                                     int(seed) & (2**64 - 1), float(eps), int(max_steps),
                                     _ptr(x), _ptr(steps), _ptr(comp))
    return x, steps, comp, int(err)


def accumulate_chunk(gi, gf, comp_side, ksqrt, pole_xy, pole_index, rep_start, rep_end,
                     seed, eps, max_steps, anchors0, blk0, blkf0, wkind0, idw_radii0,
                     idw_power0, anchors1, blk1, blkf1, wkind1, idw_radii1, idw_power1,
                     out0, out1):
    """Same contract as the reference's _kernel.accumulate_chunk (in-place +=)."""
    keep: list = []
    gi = _c(gi, np.int64)
    gf = _c(gf, np.float64)
    cs = _c(comp_side, np.int8)
    ks = _c(ksqrt, np.float64)
    pole = _c(pole_xy, np.float64)
    s0 = _side(anchors0, blk0, blkf0, wkind0, idw_radii0, idw_power0, keep)
    s1 = _side(anchors1, blk1, blkf1, wkind1, idw_radii1, idw_power1, keep)
    assert out0.flags.c_contiguous and out1.flags.c_contiguous
    stats = np.zeros(4, dtype=np.int64)
    err = lib().emo_accumulate_chunk(_ptr(gi), gi.shape[0], _ptr(gf), _ptr(cs), _ptr(ks),
                                     _ptr(pole), int(pole_index), int(rep_start),
                                     int(rep_end), int(seed) & (2**64 - 1), float(eps),
                                     int(max_steps), ctypes.byref(s0), ctypes.byref(s1),
                                     _ptr(out0), _ptr(out1), _ptr(stats))
    if err >= 0:
        return 0, 0, 0, 0, int(err)
    return int(stats[0]), int(stats[1]), int(stats[2]), int(stats[3]), -1


def run_accumulate_packed(gi, gf, comp_side, ksqrt, poles, seed, eps, max_steps, n_rep,
                          side0, side1, threads=None):
    """The reference driver (S/backend.py:147-199) over packed inputs.

    ``side0``/``side1`` are (anchors, blk, blkf, wkind, idw_radii, idw_power)
    tuples, i.e. the fields of the reference's SidePack.  Returns
    (raw0, raw1, steps_sum, steps_sq_sum, steps_max, idw_fallbacks, err) with
    err = None or (pole, replicate) of the first failing job.
    """
    keep: list = []
    gi = _c(gi, np.int64)
    gf = _c(gf, np.float64)
    cs = _c(comp_side, np.int8)
    ks = _c(ksqrt, np.float64)
    poles = _c(poles, np.float64)
    m = poles.shape[0]
    s0 = _side(*side0, keep=keep)
    s1 = _side(*side1, keep=keep)
    raw0 = np.zeros((m, s0.n_anchors))
    raw1 = np.zeros((m, s1.n_anchors))
    ss = np.zeros(m, dtype=np.int64)
    sq = np.zeros(m, dtype=np.int64)
    sm = np.zeros(m, dtype=np.int64)
    fb = np.zeros(1, dtype=np.int64)
    err = np.zeros(2, dtype=np.int64)
    threads = threads or os.cpu_count() or 1
    rc = lib().emo_run_accumulate(_ptr(gi), gi.shape[0], _ptr(gf), _ptr(cs), _ptr(ks),
                                  _ptr(poles), m, int(seed) & (2**64 - 1), float(eps),
                                  int(max_steps), int(n_rep), ctypes.byref(s0),
                                  ctypes.byref(s1), _ptr(raw0), _ptr(raw1), _ptr(ss),
                                  _ptr(sq), _ptr(sm), _ptr(fb), _ptr(err), int(threads))
    if rc < 0:
        raise MemoryError("oracle: allocation failed")
    return raw0, raw1, ss, sq, sm, int(fb[0]), (tuple(int(v) for v in err) if rc else None)


def signed_dist(gi, gf, x) -> float:
    gi = _c(gi, np.int64)
    gf = _c(gf, np.float64)
    x = _c(x, np.float64)
    return float(lib().emo_signed_dist(_ptr(gi), gi.shape[0], _ptr(gf), _ptr(x)))


def owner_component(gi, gf, x) -> int:
    gi = _c(gi, np.int64)
    gf = _c(gf, np.float64)
    x = _c(x, np.float64)
    return int(lib().emo_owner_component(_ptr(gi), gi.shape[0], _ptr(gf), _ptr(x)))


def assign_anchor(x, anchors, blk, blkf) -> int:
    keep: list = []
    s = _side(anchors, blk, blkf, keep=keep)
    x = _c(x, np.float64)
    return int(lib().emo_assign_anchor(_ptr(x), int(x.shape[0]), ctypes.byref(s)))
