"""The reference's backend boundary, B200-native.

Mirrors S/backend.py (S/ = /root/reference/pkg/src/exitmeasure/): the same
packing (``pack_geometry`` :71-83, ``pack_side`` :89-126), the same result type
(``AccumulateResult`` :137-144), the same driver entry points
(``run_accumulate`` :147-199, ``run_exits`` :202-227) and the same chunk
contract of the ``_impl`` module (``walk_exits_chunk`` / ``accumulate_chunk``,
S/_kernel.pyx:376-464) -- but every walk runs in ONE launch of a CUDA kernel
(libexitmeasure_b200.so) instead of a thread pool over 8192-walk chunks.

Two arithmetic paths (``precision``):

* ``"ref64"`` (default): the bit-exact FP64 mirror -- identical counts,
  exits and step statistics to the reference kernel for the same inputs.
* ``"fp32"``: the production kernel (Philox4x32 streams, FP32 state, O(1)
  binning); statistically identical exit law, not bit-identical.  With
  ``chain="max"`` each step uses the largest certified K^{1/2}-ellipsoid
  instead of the reference's sd-scaled one (fewer steps, same stopping shell
  and exit law); ``chain="tangent"`` (default for fp32) walks on balls that
  touch the boundary near the current point in whitened coordinates -- the
  largest ball tangent to the nearest face (2D / 3D boxes, the L-box), balls
  rolling inside the whitened ellipse / ellipsoid and disks tangent to a
  concentric hole (ball, annulus) -- sampling each ball's harmonic measure
  exactly (quadratic approach to the boundary), and runs "max" elsewhere
  (K = I, non-concentric holes).

``EXITMEASURE_B200_PRECISION`` / ``EXITMEASURE_B200_CHAIN`` set the defaults
process-wide (the analogue of the reference's ``EXITMEASURE_BACKEND``).
There is no CPU fallback: a missing library or device raises NativeError.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
import weakref
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NativeError, ValidationError, WalkBudgetError

BACKEND = "cuda"
CHUNK = 8192  # kept for API parity (S/backend.py:43-45); the GPU path does not chunk

_WEIGHT_KINDS = {"voronoi": 0, "idw": 1}
_BLOCK_KIND = {"generic": 0, "circle": 1, "square": 2, "sphere": 0}
_PRECISIONS = {"ref64": N.EM_PREC_REF64, "fp64": N.EM_PREC_REF64, "exact": N.EM_PREC_REF64,
               "fp32": N.EM_PREC_FP32}
_CHAINS = {"woe": N.EM_CHAIN_WOE, "reference": N.EM_CHAIN_WOE, "max": N.EM_CHAIN_MAX,
           "tangent": N.EM_CHAIN_TANGENT}
_CHAIN_NAMES = {N.EM_CHAIN_WOE: "woe", N.EM_CHAIN_MAX: "max", N.EM_CHAIN_TANGENT: "tangent"}


def default_precision() -> str:
    return os.environ.get("EXITMEASURE_B200_PRECISION", "ref64").lower()


def default_chain(precision: str) -> str:
    env = os.environ.get("EXITMEASURE_B200_CHAIN")
    if env:
        return env.lower()
    return "woe" if _PRECISIONS[precision] == N.EM_PREC_REF64 else "tangent"


def resolve_chain(geom: "GeomPack", ksqrt, precision: str | None = None,
                  chain: str | None = None) -> str:
    """The chain a plan over ``geom`` runs for (precision, chain) -- "tangent"
    becomes "max" where the geometry has no tangent-ball step (em_resolve_chain;
    no device needed)."""
    precision = (precision or default_precision()).lower()
    chain = (chain or default_chain(precision)).lower()
    if precision not in _PRECISIONS:
        raise ValidationError(f"unknown precision {precision!r}")
    if chain not in _CHAINS:
        raise ValidationError(f"unknown chain {chain!r}")
    m = _Marshal()
    g = m.geometry(geom.gi, geom.gf, geom.comp_side, ksqrt)
    rc = N.lib().em_resolve_chain(N.ctypes.byref(g), _PRECISIONS[precision], _CHAINS[chain])
    N.check(rc, "em_resolve_chain")
    return _CHAIN_NAMES[rc]


def f32_constant(geom: "GeomPack", ksqrt, chain: str, eps: float, name: str,
                 ident: bool = False) -> np.ndarray:
    """One closed-form constant of the FP32 kernel for this geometry and
    (resolved) chain, as em_plan_create computes it -- host only, no device
    (em_f32_constant; the host unit tests of the plan constants)."""
    m = _Marshal()
    g = m.geometry(geom.gi, geom.gf, geom.comp_side, ksqrt)
    out = np.zeros(128, dtype=np.float32)
    k = N.lib().em_f32_constant(ctypes.byref(g), _CHAINS[chain], int(ident), float(eps),
                                name.encode(), N.ptr(out), out.size)
    if k < 0:
        raise ValidationError(f"unknown FP32 constant {name!r}")
    return out[:k].copy()


def default_device() -> int:
    return int(os.environ.get("EXITMEASURE_B200_DEVICE", "0"))


@dataclass(frozen=True, eq=False)
class GeomPack:
    gi: np.ndarray  # int64 [d, outer_kind, n_holes(, n_notch)]
    gf: np.ndarray  # float64 [outer..., holes..., (nx, ny)]
    comp_side: np.ndarray  # int8 per component: 0 gamma0, 1 gamma1


@dataclass(frozen=True, eq=False)
class SidePack:
    anchors: np.ndarray  # (M, d) float64
    blk: np.ndarray  # (B, 3) int64: kind, start, count
    blkf: np.ndarray  # (B, 4) float64: cx, cy, cz, radius
    weights_kind: int
    idw_radii: np.ndarray
    idw_power: int
    blk_phase: np.ndarray | None = None  # (B,) extension: anchor phase per block

    @property
    def size(self) -> int:
        return self.anchors.shape[0]


def _is_ball(shape) -> bool:
    return hasattr(shape, "radius") and not hasattr(shape, "halfwidth")


def pack_geometry(dom) -> GeomPack:
    """S/backend.py:71-83, plus the L-box notch as gi[3] = 1 (duck-typed:
    works on the reference's Domain objects too)."""
    d = int(dom.dimension)
    outer = dom.outer
    outer_kind = 0 if _is_ball(outer) else 1
    notch = getattr(outer, "notch", None)
    gi = [d, outer_kind, len(dom.holes)] + ([1] if notch is not None else [])
    parts = list(np.asarray(outer.center, dtype=float))
    parts.append(float(outer.radius if outer_kind == 0 else outer.halfwidth))
    for h in dom.holes:
        parts.extend(np.asarray(h.center, dtype=float))
        parts.append(float(h.radius))
    if notch is not None:
        parts.extend([float(notch[0]), float(notch[1])])
    n_comp = 1 + len(dom.holes) + (1 if notch is not None else 0)
    side = np.array([0 if c in dom.gamma0 else 1 for c in range(n_comp)], dtype=np.int8)
    return GeomPack(np.asarray(gi, dtype=np.int64), np.asarray(parts, dtype=np.float64), side)


def pack_side(anchors, d: int, eps: float, weights_kind: str = "voronoi",
              idw_radii: np.ndarray | None = None, idw_power: int = 2) -> SidePack:
    """S/backend.py:89-126 (same block kinds, same square-pruning gate, same
    brute-force fallback for uncovered anchors) plus per-block phases."""
    if anchors is None or len(anchors) == 0:
        return SidePack(np.zeros((0, d)), np.zeros((1, 3), dtype=np.int64),
                        np.zeros((1, 4)), 0, np.zeros(0), 2, np.zeros(1))
    pts = np.ascontiguousarray(anchors.points, dtype=np.float64)
    blocks = anchors.blocks or ()
    blk, blkf, phase = [], [], []
    covered = 0
    for b in blocks:
        kind = _BLOCK_KIND.get(b.kind, 0) if b.uniform else 0
        if kind == 2:
            spacing = 8.0 * b.radius / b.count
            if eps > spacing / 16.0:
                kind = 0
        blk.append((kind, b.start, b.count))
        c3 = np.zeros(3)
        c3[: np.asarray(b.center).shape[0]] = b.center
        blkf.append((c3[0], c3[1], c3[2], b.radius))
        phase.append(float(getattr(b, "phase", 0.0)) if kind in (1, 2) else 0.0)
        covered += b.count
    if covered != len(anchors):
        blk = [(0, 0, len(anchors))]
        blkf = [(0.0, 0.0, 0.0, 0.0)]
        phase = [0.0]
    wk = _WEIGHT_KINDS[weights_kind]
    if wk == 1:
        if idw_radii is None or idw_radii.shape[0] != len(anchors):
            raise ValidationError("idw radii must match the anchor count")
        radii = np.ascontiguousarray(idw_radii, dtype=np.float64)
    else:
        radii = np.zeros(0)
    return SidePack(pts, np.asarray(blk, dtype=np.int64), np.asarray(blkf, dtype=np.float64),
                    wk, radii, int(idw_power), np.asarray(phase, dtype=np.float64))


# ---------------------------------------------------------------------------
# ctypes marshalling (keeps the numpy buffers alive for the call)


class _Marshal:
    def __init__(self):
        self.keep = []

    def arr(self, a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        self.keep.append(a)
        return a

    def geometry(self, gi, gf, comp_side, ksqrt) -> N.EmGeometry:
        gi = self.arr(gi, np.int64)
        gf = self.arr(gf, np.float64)
        cs = self.arr(comp_side, np.int8)
        ks = self.arr(ksqrt, np.float64)
        d = int(gi[0])
        if ks.size != d * d:
            raise ValidationError(f"ksqrt must be {d}x{d}")
        return N.EmGeometry(N.ptr(gi), gi.shape[0], N.ptr(gf), gf.shape[0], N.ptr(cs),
                            cs.shape[0], N.ptr(ks))

    def side(self, anchors, blk, blkf, wkind, idw_radii, idw_power, phase=None) -> N.EmSide:
        anchors = self.arr(anchors, np.float64)
        blk = self.arr(blk, np.int64).reshape(-1, 3)
        blkf = self.arr(blkf, np.float64).reshape(-1, 4)
        radii = self.arr(idw_radii if idw_radii is not None else np.zeros(0), np.float64)
        ph = None if phase is None else self.arr(phase, np.float64)
        return N.EmSide(N.ptr(anchors), anchors.shape[0], N.ptr(blk), N.ptr(blkf), blk.shape[0],
                        int(wkind), int(idw_power), N.ptr(radii),
                        N.ptr(ph) if ph is not None else None)

    def sidepack(self, sp) -> N.EmSide:
        return self.side(sp.anchors, sp.blk, sp.blkf, sp.weights_kind, sp.idw_radii,
                         sp.idw_power, getattr(sp, "blk_phase", None))


def _has_idw(*sides) -> bool:
    return any(int(getattr(s, "weights_kind", 0)) != 0 for s in sides)


# ---------------------------------------------------------------------------
# the _impl chunk contract (S/_kernel.pyx:376-464), bit-exact REF64


def walk_exits_chunk(gi, gf, comp_side, ksqrt, pole_xy, pole_index, rep_start, rep_end, seed,
                     eps, max_steps, device: int | None = None):
    """Drop-in for _kernel.walk_exits_chunk: (x (n,d), steps, comp, err)."""
    m = _Marshal()
    g = m.geometry(gi, gf, comp_side, ksqrt)
    pole = m.arr(pole_xy, np.float64)
    d = int(np.asarray(gi)[0])
    n = int(rep_end) - int(rep_start)
    x = np.empty((n, d))
    steps = np.empty(n, dtype=np.int64)
    comp = np.empty(n, dtype=np.int64)
    err = ctypes.c_int64(-1)
    dev = default_device() if device is None else device
    N.check(N.lib().em_walk_exits_chunk(ctypes.byref(g), N.ptr(pole), int(pole_index),
                                        int(rep_start), int(rep_end),
                                        int(seed) & (2**64 - 1), float(eps), int(max_steps),
                                        dev, N.ptr(x), N.ptr(steps), N.ptr(comp),
                                        ctypes.byref(err)), "em_walk_exits_chunk")
    return x, steps, comp, int(err.value)


def accumulate_chunk(gi, gf, comp_side, ksqrt, pole_xy, pole_index, rep_start, rep_end, seed,
                     eps, max_steps, anchors0, blk0, blkf0, wkind0, idw_radii0, idw_power0,
                     anchors1, blk1, blkf1, wkind1, idw_radii1, idw_power1, out0, out1,
                     device: int | None = None):
    """Drop-in for _kernel.accumulate_chunk: out0/out1 += counts; returns
    (steps_sum, steps_sq_sum, steps_max, idw_fallbacks, err)."""
    m = _Marshal()
    g = m.geometry(gi, gf, comp_side, ksqrt)
    pole = m.arr(pole_xy, np.float64)
    s0 = m.side(anchors0, blk0, blkf0, wkind0, idw_radii0, idw_power0)
    s1 = m.side(anchors1, blk1, blkf1, wkind1, idw_radii1, idw_power1)
    if not (out0.flags.c_contiguous and out1.flags.c_contiguous):
        raise ValidationError("out0/out1 must be C-contiguous float64")
    stats = np.zeros(4, dtype=np.int64)
    err = ctypes.c_int64(-1)
    dev = default_device() if device is None else device
    N.check(N.lib().em_accumulate_chunk(ctypes.byref(g), N.ptr(pole), int(pole_index),
                                        int(rep_start), int(rep_end),
                                        int(seed) & (2**64 - 1), float(eps), int(max_steps),
                                        ctypes.byref(s0), ctypes.byref(s1), dev,
                                        N.ptr(out0), N.ptr(out1), N.ptr(stats),
                                        ctypes.byref(err)), "em_accumulate_chunk")
    if err.value >= 0:
        return 0, 0, 0, 0, int(err.value)
    return int(stats[0]), int(stats[1]), int(stats[2]), int(stats[3]), -1


# ---------------------------------------------------------------------------
# batched driver


class AccumulateResult:
    """Per-pole exit rows of a run (S/backend.py:137-144's fields).

    ``counts`` holds the exact int64 rows (side-0 columns first); ``raw0`` /
    ``raw1`` are the reference's float64 views of them, converted on first
    access (IDW runs set them directly: their rows are fractional)."""

    def __init__(self, raw0=None, raw1=None, steps_sum=None, steps_sq_sum=None, steps_max=None,
                 idw_fallbacks: int = 0, counts=None, kernel_ms: float = 0.0, n0: int | None = None):
        self._raw0, self._raw1 = raw0, raw1
        self.steps_sum = steps_sum
        self.steps_sq_sum = steps_sq_sum
        self.steps_max = steps_max
        self.idw_fallbacks = idw_fallbacks
        self.counts = counts
        self.kernel_ms = kernel_ms
        self._n0 = n0 if n0 is not None else (raw0.shape[1] if raw0 is not None else 0)

    @property
    def raw0(self) -> np.ndarray:
        if self._raw0 is None:
            self._raw0 = self.counts[:, : self._n0].astype(np.float64)
        return self._raw0

    @property
    def raw1(self) -> np.ndarray:
        if self._raw1 is None:
            self._raw1 = self.counts[:, self._n0:].astype(np.float64)
        return self._raw1


def _free_block(addr: int) -> None:
    N.lib().em_host_block_free(ctypes.c_void_p(addr))


class Plan:
    """One problem resident on one GPU: geometry, K^{1/2}, poles, both weight
    families (and their binning accelerators) uploaded once; ``run`` walks
    replicates [rep_start, rep_start + n_rep) of every pole in one launch.

    ``pole_ids`` are the pole indices that key the RNG streams (default
    0..M-1); a row shard passes its global indices so that sharded runs
    reproduce the single-GPU counts exactly.
    """

    def __init__(self, geom: GeomPack, ksqrt, poles, eps: float, max_steps: int,
                 side0, side1, precision: str | None = None, chain: str | None = None,
                 device: int | None = None, pole_ids=None, block: int = 0, grid: int = 0,
                 flags: int = 0):
        precision = (precision or default_precision()).lower()
        if precision not in _PRECISIONS:
            raise ValidationError(f"unknown precision {precision!r}")
        chain = (chain or default_chain(precision)).lower()
        if chain not in _CHAINS:
            raise ValidationError(f"unknown chain {chain!r}")
        self.idw = _has_idw(side0, side1)
        self.device = default_device() if device is None else int(device)
        N.require_device(self.device)
        self.precision, self.chain = precision, chain
        self.d = int(geom.gi[0])
        self.poles = np.ascontiguousarray(poles, dtype=np.float64).reshape(-1, self.d)
        self.n_poles = self.poles.shape[0]
        self.n0, self.n1 = int(side0.size), int(side1.size)
        m = _Marshal()
        g = m.geometry(geom.gi, geom.gf, geom.comp_side, ksqrt)
        s0 = m.sidepack(side0)
        s1 = m.sidepack(side1)
        pl = m.arr(self.poles, np.float64)
        pid = None if pole_ids is None else m.arr(pole_ids, np.int64)
        if pid is not None and pid.shape[0] != self.n_poles:
            raise ValidationError("one pole id per pole required")
        # budget errors name the GLOBAL pole (the RNG key), as the reference's
        # job-order scan does (S/backend.py:189-192)
        self.pole_ids = None if pid is None else pid.copy()
        opt = N.EmOptions(_PRECISIONS[precision], _CHAINS[chain], self.device, int(block),
                          int(grid), int(flags))
        h = ctypes.c_void_p()
        N.check(N.lib().em_plan_create(ctypes.byref(g), ctypes.byref(s0), ctypes.byref(s1),
                                       N.ptr(pl), N.ptr(pid) if pid is not None else None,
                                       self.n_poles, float(eps), int(max_steps),
                                       ctypes.byref(opt), ctypes.byref(h)), "em_plan_create")
        self._h = h
        self.max_steps = int(max_steps)
        # the chain the plan runs: "tangent" becomes "max" where the geometry
        # has no tangent-ball step (em_plan_chain)
        self.chain = _CHAIN_NAMES.get(int(N.lib().em_plan_chain(h)), chain)

    def _budget_error(self, row: int, replicate: int) -> WalkBudgetError:
        """WalkBudgetError for plan row ``row``, naming its global pole id."""
        pole = int(self.pole_ids[row]) if self.pole_ids is not None else int(row)
        return WalkBudgetError(pole, int(replicate), self.max_steps)

    def close(self):
        if getattr(self, "_h", None):
            N.lib().em_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def run_raw(self, seed: int, n_rep: int, rep_start: int = 0,
                chunk: int = CHUNK) -> AccumulateResult:
        """Fractional rows (IDW families), summed with the reference driver's
        per-CHUNK partials in job order -- bit-identical rows on REF64; on
        FP32 the same fixed-order FP64 weights over the FP32 kernel's exits."""
        raw0 = np.zeros((self.n_poles, self.n0))
        raw1 = np.zeros((self.n_poles, self.n1))
        stats = np.zeros((3, self.n_poles), dtype=np.int64)
        fb, ep, er = ctypes.c_int64(0), ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = N.check(N.lib().em_plan_run_raw(self._h, int(seed) & (2**64 - 1), int(rep_start),
                                             int(n_rep), int(chunk), None, None, N.ptr(raw0),
                                             N.ptr(raw1), N.ptr(stats), ctypes.byref(fb),
                                             ctypes.byref(ep), ctypes.byref(er)),
                     "em_plan_run_raw")
        if rc == N.EM_BUDGET:
            raise self._budget_error(ep.value, rep_start + er.value)
        return AccumulateResult(raw0, raw1, stats[0].copy(), stats[1].copy(), stats[2].copy(),
                                int(fb.value))

    def run(self, seed: int, n_rep: int, rep_start: int = 0,
            rows: str = "int64") -> AccumulateResult:
        """All walks of the plan; ``rows="float64"`` returns the reference's
        float64 raw0 / raw1 converted on the device (em_plan_run_host_f64,
        no host-side conversion; ``counts`` is then None)."""
        if self.idw:
            return self.run_raw(seed, n_rep, rep_start)
        if rows not in ("int64", "float64"):
            raise ValidationError("rows must be 'int64' or 'float64'")
        row = self.n0 + self.n1
        blk = ctypes.POINTER(ctypes.c_int64)()
        ep, er = ctypes.c_int64(-1), ctypes.c_int64(-1)
        fn = N.lib().em_plan_run_host_f64 if rows == "float64" else N.lib().em_plan_run_host
        rc = N.check(fn(self._h, int(seed) & (2**64 - 1), int(rep_start), int(n_rep),
                        ctypes.byref(blk), ctypes.byref(ep), ctypes.byref(er)),
                     "em_plan_run_host")
        if rc == N.EM_BUDGET:
            raise self._budget_error(ep.value, rep_start + er.value)
        nc = self.n_poles * row
        # zero-copy: the result owns the page-locked block the counts were
        # copied into (returned to the library's cache when the arrays die)
        N.check(N.lib().em_plan_detach_block(self._h, ctypes.byref(blk)), "em_plan_detach_block")
        addr = ctypes.cast(blk, ctypes.c_void_p).value
        cbuf = (ctypes.c_int64 * (nc + 3 * self.n_poles)).from_address(addr)
        weakref.finalize(cbuf, _free_block, addr)  # every numpy view keeps cbuf alive
        view = np.frombuffer(cbuf, dtype=np.int64)
        stats = view[nc:].reshape(3, self.n_poles)
        ms = ctypes.c_double(0)
        N.lib().em_plan_last_stats(self._h, ctypes.byref(ms), None, None)
        if rows == "float64":
            f = np.frombuffer(cbuf, dtype=np.float64, count=nc).reshape(self.n_poles, row)
            return AccumulateResult(f[:, : self.n0], f[:, self.n0:], stats[0], stats[1],
                                    stats[2], 0, None, ms.value, n0=self.n0)
        counts = view[:nc].reshape(self.n_poles, row)
        return AccumulateResult(None, None, stats[0], stats[1], stats[2], 0, counts, ms.value,
                                n0=self.n0)

    def run_device(self, seed: int, n_rep: int, counts_ptr: int, stats_ptr: int,
                   stream_ptr: int | None = None, rep_start: int = 0) -> None:
        """Outputs stay in device memory: counts (n_poles, n0+n1) int64 and
        stats (3, n_poles) int64 at the given device pointers; work is
        ordered on ``stream_ptr`` (e.g. torch's current stream) and this call
        returns without waiting -- call ``check()`` after synchronising.
        Integer rows only: IDW families need ``run_raw``."""
        if self.idw:
            raise ValidationError("IDW weight families give fractional rows: use run_raw")
        out = N.EmOutputs(ctypes.c_void_p(counts_ptr), ctypes.c_void_p(stats_ptr),
                          ctypes.c_void_p(stats_ptr + 8 * self.n_poles),
                          ctypes.c_void_p(stats_ptr + 16 * self.n_poles), -1, -1)
        # torch reports the legacy default stream as handle 0, which this ABI
        # reads as "the plan's own stream": pass cudaStreamLegacy (0x1) instead
        # so the work is ordered with the caller's events and kernels
        sp = stream_ptr if stream_ptr else 1
        N.check(N.lib().em_plan_run_device(self._h, int(seed) & (2**64 - 1), int(rep_start),
                                           int(n_rep), ctypes.byref(out), ctypes.c_void_p(sp)),
                "em_plan_run_device")
        self._last_rep_start = int(rep_start)

    def check(self) -> None:
        """Raise WalkBudgetError if the last run_device hit the step budget
        (waits for the plan's stream)."""
        ep, er = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = N.check(N.lib().em_plan_check(self._h, ctypes.byref(ep), ctypes.byref(er)),
                     "em_plan_check")
        if rc == N.EM_BUDGET:
            raise self._budget_error(ep.value, getattr(self, "_last_rep_start", 0) + er.value)

    def exits(self, seed: int, n_rep: int, rep_start: int = 0):
        """Exit points, steps and components of n_rep walks per pole,
        (pole, replicate)-major."""
        total = self.n_poles * int(n_rep)
        x = np.empty((total, self.d))
        steps = np.empty(total, dtype=np.int64)
        comp = np.empty(total, dtype=np.int64)
        ep, er = ctypes.c_int64(-1), ctypes.c_int64(-1)
        rc = N.check(N.lib().em_run_exits(self._h, int(seed) & (2**64 - 1), int(rep_start),
                                          int(n_rep), N.ptr(x), N.ptr(steps), N.ptr(comp),
                                          ctypes.byref(ep), ctypes.byref(er)), "em_run_exits")
        if rc == N.EM_BUDGET:
            raise self._budget_error(ep.value, rep_start + er.value)
        return x, steps, comp

    def bin_points(self, pts):
        """(component, side, anchor index) of each point under the plan's
        binning rule (owner component -> side -> nearest anchor)."""
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, self.d)
        n = pts.shape[0]
        comp = np.empty(n, dtype=np.int64)
        side = np.empty(n, dtype=np.int64)
        bins = np.empty(n, dtype=np.int64)
        N.check(N.lib().em_bin_points(self._h, N.ptr(pts), n, N.ptr(comp), N.ptr(side),
                                      N.ptr(bins)), "em_bin_points")
        return comp, side, bins

    def debug_step(self, x, words):
        """ONE step of the plan's FP32 chain from each world point x (n, d)
        with random words (n, 2) uint32 (em_debug_step): (candidate next
        points (n, d), 0/1 stop masks at x)."""
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, self.d)
        w = np.ascontiguousarray(words, dtype=np.uint32).reshape(-1, 2)
        if w.shape[0] != x.shape[0]:
            raise ValidationError("one word pair per point")
        y = np.empty_like(x)
        mask = np.empty(x.shape[0], dtype=np.float32)
        N.check(N.lib().em_debug_step(self._h, N.ptr(x), N.ptr(w), x.shape[0], N.ptr(y),
                                      N.ptr(mask)), "em_debug_step")
        return y, mask

    def last_stats(self):
        ms = ctypes.c_double(0)
        w = ctypes.c_int64(0)
        s = ctypes.c_int64(0)
        N.lib().em_plan_last_stats(self._h, ctypes.byref(ms), ctypes.byref(w), ctypes.byref(s))
        return ms.value, w.value, s.value

    def last_scheduler(self) -> str:
        """Scheduler of the last integer-count run (em_plan_last_scheduler)."""
        return {0: "persistent", 1: "persistent+smem-stats", 2: "pole-blocks"}.get(
            int(N.lib().em_plan_last_scheduler(self._h)), "none")

    def walks_per_lane(self) -> int:
        """2 where counts run on the packed two-walks-per-lane kernel."""
        return int(N.lib().em_plan_walks_per_lane(self._h))

    def last_walks_per_lane(self) -> int:
        """Walks per lane of the last integer-count run (small runs take the
        one-walk kernel unless EM_FLAG_TWO_WALKS_PER_LANE)."""
        return int(N.lib().em_plan_last_walks_per_lane(self._h))

    def last_launches(self) -> int:
        v = ctypes.c_int64(0)
        N.lib().em_plan_last_launches(self._h, ctypes.byref(v))
        return int(v.value)


# Plans of recent run_accumulate calls, keyed by the content of every input
# that shapes the plan (geometry, K, poles, pole ids, both sides, eps, budget,
# precision, chain, device): a repeated call with the same inputs (a parameter
# sweep over seeds or walk counts, the reference's benchmark loop) skips plan
# creation and the input upload.  Results are detached from the plan, so a
# cached plan is reusable as soon as run() returns; a plan busy in another
# thread is bypassed with a one-shot plan.
_PLAN_CACHE: "OrderedDict[tuple, tuple[Plan, threading.Lock]]" = OrderedDict()
_PLAN_CACHE_LOCK = threading.Lock()
_PLAN_CACHE_SIZE = 4


def _plan_key(geom, ksqrt, poles, eps, max_steps, side0, side1, precision, chain, device,
              pole_ids) -> tuple:
    """(scalars + dtypes/shapes, concatenated array bytes): the plan's full
    input content, compared exactly (no digest: ~5 us for cfg2's 12 KiB)."""
    arrays = (geom.gi, geom.gf, geom.comp_side, ksqrt, poles, pole_ids,
              side0.anchors, side0.blk, side0.blkf, side0.idw_radii, getattr(side0, "blk_phase", None),
              side1.anchors, side1.blk, side1.blkf, side1.idw_radii, getattr(side1, "blk_phase", None))
    # the reference's own SidePack (plugin path) has the same fields minus blk_phase
    meta = [float(eps), int(max_steps), int(side0.weights_kind), int(side0.idw_power),
            int(side1.weights_kind), int(side1.idw_power), precision, chain, device]
    parts = []
    for a in arrays:
        if a is None:
            meta.append(None)
        else:
            a = np.asarray(a)
            meta.append((a.dtype.str, a.shape))
            parts.append(a.tobytes())
    return tuple(meta), b"".join(parts)


def run_accumulate(dom, ksqrt, poles, seed: int, eps: float, max_steps: int, n_rep: int,
                   side0, side1, threads: int | None = None, *, precision: str | None = None,
                   chain: str | None = None, device: int | None = None,
                   pole_ids=None, cache: bool = True, rows: str = "int64") -> AccumulateResult:
    """All (pole, replicate) walks in one kernel launch (S/backend.py:147-199).

    ``cache=False`` builds (and uploads) a one-shot plan even when a cached
    plan for the same inputs exists.  ``rows="float64"`` converts the rows
    to the reference's float64 raw0 / raw1 on the device (``counts`` None).

    ``threads`` is accepted for signature compatibility and ignored.  Raises
    WalkBudgetError(pole, replicate, max_steps) for the lexicographically
    first failing walk, like the reference's job-order scan.
    """
    geom = pack_geometry(dom)
    poles = np.ascontiguousarray(poles, dtype=np.float64)
    if poles.ndim == 1:
        poles = poles.reshape(1, -1)
    if poles.shape[0] == 0:  # no jobs: the reference returns empty rows (S/backend.py:150-199)
        z = np.zeros(0, dtype=np.int64)
        return AccumulateResult(np.zeros((0, int(side0.size))), np.zeros((0, int(side1.size))),
                                z, z.copy(), z.copy(), 0, np.zeros((0, int(side0.size + side1.size)),
                                                                   dtype=np.int64),
                                n0=int(side0.size))
    precision = (precision or default_precision()).lower()
    chain = (chain or default_chain(precision)).lower()
    device = default_device() if device is None else int(device)
    if not cache:
        with Plan(geom, ksqrt, poles, eps, max_steps, side0, side1, precision, chain, device,
                  pole_ids) as plan:
            return plan.run(seed, n_rep, rows=rows)
    key = _plan_key(geom, ksqrt, poles, eps, max_steps, side0, side1, precision, chain, device,
                    pole_ids)
    with _PLAN_CACHE_LOCK:
        hit = _PLAN_CACHE.get(key)
        if hit is not None:
            _PLAN_CACHE.move_to_end(key)
    if hit is not None and hit[1].acquire(blocking=False):
        try:
            return hit[0].run(seed, n_rep, rows=rows)
        finally:
            hit[1].release()
    plan = Plan(geom, ksqrt, poles, eps, max_steps, side0, side1, precision, chain, device,
                pole_ids)
    lock = threading.Lock()
    with lock:
        res = plan.run(seed, n_rep, rows=rows)
    if hit is None:
        with _PLAN_CACHE_LOCK:
            if key not in _PLAN_CACHE:
                _PLAN_CACHE[key] = (plan, lock)
                while len(_PLAN_CACHE) > _PLAN_CACHE_SIZE:
                    _PLAN_CACHE.popitem(last=False)
                return res
    plan.close()
    return res


def clear_plan_cache() -> None:
    """Release the plans cached by run_accumulate."""
    with _PLAN_CACHE_LOCK:
        items = list(_PLAN_CACHE.values())
        _PLAN_CACHE.clear()
    for plan, lock in items:
        with lock:
            plan.close()


def run_exits(dom, ksqrt, pole_xy, pole_index: int, seed: int, eps: float, max_steps: int,
              n_rep: int, threads: int | None = None, *, precision: str | None = None,
              chain: str | None = None, device: int | None = None):
    """Exit points, step counts and owning components for one pole
    (S/backend.py:202-227)."""
    geom = pack_geometry(dom)
    d = int(geom.gi[0])
    pole = np.ascontiguousarray(pole_xy, dtype=np.float64).reshape(1, d)
    precision = (precision or default_precision()).lower()
    if _PRECISIONS.get(precision) == N.EM_PREC_REF64:
        x, steps, comp, err = walk_exits_chunk(geom.gi, geom.gf, geom.comp_side, ksqrt,
                                               pole[0], pole_index, 0, n_rep, seed, eps,
                                               max_steps, device)
        if err >= 0:
            raise WalkBudgetError(pole_index, err, max_steps)
        return x, steps, comp
    # the FP32 exits kernel: any side needs >=1 anchor for plan validation
    dummy = SidePack(np.zeros((1, d)), np.array([[0, 0, 1]], dtype=np.int64), np.zeros((1, 4)),
                     0, np.zeros(0), 2, np.zeros(1))
    cs = np.zeros_like(geom.comp_side)
    g2 = GeomPack(geom.gi, geom.gf, cs)
    with Plan(g2, ksqrt, pole, eps, max_steps, dummy, dummy, precision, chain, device,
              np.array([pole_index], dtype=np.int64)) as plan:
        try:
            return plan.exits(seed, n_rep)
        except WalkBudgetError as e:
            raise WalkBudgetError(pole_index, e.replicate, max_steps) from None


def is_available(device: int = 0) -> bool:
    try:
        return N.device_count() > device
    except NativeError:
        return False
