"""Domain, boundary point-set and anchor-block types for the exit-measure path.

Mirrors the reference's geometry model (S/geometry.py:26-135, S/ =
/root/reference/pkg/src/exitmeasure/) with the same field names, so objects
built by the reference package can be passed to this package's backend
unchanged (the packers duck-type on ``radius`` / ``halfwidth`` / ``notch``).

Extensions the BASELINE configs need and the reference cannot express
(SURVEY.md Appendix A):

* ``LBox`` -- the box [c-h, c+h]^3 minus the quadrant prism {x >= nx, y >= ny}
  (cfg5's L-shaped box).  Its boundary components are 0 (outer box faces) and
  ``1 + n_holes`` (the two notch faces meeting at the re-entrant edge).
* ``AnchorBlock.phase`` -- a uniform circle/square block whose anchors sit at
  ``spacing * (k + phase)`` along the curve (phase 0 is the reference layout
  of ``circle_points`` / ``square_points``; 0.5 puts anchors at cell
  midpoints, the layout of cfg1/cfg2's arc and edge bins).
* ``AnchorBlock.kind == "grid"`` is never user-facing; generic blocks are
  accelerated by a candidate grid built inside the native library.

Component ids: 0 is the outer boundary, 1..L the ball holes in order, L+1 the
notch (when present).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .errors import ValidationError

GAMMA0 = "gamma0"
GAMMA1 = "gamma1"


@dataclass(frozen=True, eq=False)
class Ball:
    center: np.ndarray
    radius: float

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=float))
        if self.radius <= 0:
            raise ValidationError(f"ball radius must be positive, got {self.radius}")


@dataclass(frozen=True, eq=False)
class Box:
    """Axis-aligned cube [-h, h]^d shifted to ``center`` (S/geometry.py:37-47)."""

    center: np.ndarray
    halfwidth: float

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=float))
        if self.halfwidth <= 0:
            raise ValidationError(f"box halfwidth must be positive, got {self.halfwidth}")


@dataclass(frozen=True, eq=False)
class LBox:
    """Box minus the quadrant prism {x >= notch[0], y >= notch[1]} (3D only).

    BASELINE cfg5: center (.5,.5,.5), halfwidth .5, notch (.5, .5) gives
    [0,1]^3 minus [.5,1]^2 x [0,1].
    """

    center: np.ndarray
    halfwidth: float
    notch: tuple

    def __post_init__(self):
        object.__setattr__(self, "center", np.asarray(self.center, dtype=float))
        object.__setattr__(self, "notch", tuple(float(v) for v in self.notch))
        c, h = self.center, self.halfwidth
        if h <= 0:
            raise ValidationError("box halfwidth must be positive")
        if len(self.notch) != 2:
            raise ValidationError("notch is the (x, y) corner of the removed prism")
        for j in range(2):
            if not (c[j] - h < self.notch[j] < c[j] + h):
                raise ValidationError("notch corner must lie strictly inside the box")


@dataclass(frozen=True, eq=False)
class Domain:
    dimension: int
    outer: object
    holes: tuple = ()
    gamma0: frozenset = frozenset()

    def __post_init__(self):
        object.__setattr__(self, "gamma0", frozenset(self.gamma0))
        object.__setattr__(self, "holes", tuple(self.holes))
        d = self.dimension
        if d not in (2, 3):
            raise ValidationError(f"dimension must be 2 or 3, got {d}")
        if self.outer.center.shape != (d,):
            raise ValidationError("outer shape dimension mismatch")
        if isinstance(self.outer, LBox) and d != 3:
            raise ValidationError("the L-box is a 3D domain")
        for h in self.holes:
            if h.center.shape != (d,):
                raise ValidationError("hole dimension mismatch")
        bad = self.gamma0 - set(range(self.n_components))
        if bad:
            raise ValidationError(f"gamma0 references unknown components {sorted(bad)}")

    @property
    def has_notch(self) -> bool:
        return hasattr(self.outer, "notch")

    @property
    def n_components(self) -> int:
        return 1 + len(self.holes) + (1 if self.has_notch else 0)

    @property
    def gamma1(self) -> frozenset:
        return frozenset(range(self.n_components)) - self.gamma0

    def side_of(self, component: int) -> str:
        return GAMMA0 if component in self.gamma0 else GAMMA1


def make_domain(outer, holes=(), gamma0=(0,)) -> Domain:
    d = np.asarray(outer.center).shape[0]
    return Domain(d, outer, tuple(holes), frozenset(gamma0))


@dataclass(frozen=True, eq=False)
class AnchorBlock:
    """One structured run of anchors (S/geometry.py:107-124) + ``phase``."""

    kind: str
    start: int
    count: int
    component: int
    center: np.ndarray
    radius: float
    uniform: bool = True
    phase: float = 0.0


@dataclass(frozen=True, eq=False)
class BoundaryPointSet:
    points: np.ndarray
    component_ids: np.ndarray
    params: np.ndarray
    blocks: tuple = field(default=())

    def __len__(self) -> int:
        return self.points.shape[0]


# ---------------------------------------------------------------------------
# signed distance (host-side validation; the walk itself runs on the GPU)


def _norm(v) -> float:
    t = v[0] * v[0] + v[1] * v[1]
    if v.shape[0] == 3:
        t = t + v[2] * v[2]
    return math.sqrt(t)


def _outer_signed(shape, x) -> float:
    if hasattr(shape, "radius"):
        return shape.radius - _norm(x - shape.center)
    q = np.abs(x - shape.center) - shape.halfwidth
    m = float(np.max(q))
    if m <= 0.0:
        return -m
    return -_norm(np.maximum(q, 0.0))


def notch_signed(notch, x) -> float:
    """Signed distance to the notch prism, positive outside it (em_oracle.c)."""
    qx = notch[0] - x[0]
    qy = notch[1] - x[1]
    if qx <= 0.0 and qy <= 0.0:
        return max(qx, qy)
    ax, ay = max(qx, 0.0), max(qy, 0.0)
    return math.sqrt(ax * ax + ay * ay)


def dist_to_boundary(dom, x) -> float:
    """Signed Euclidean distance to the whole boundary (S/geometry.py:172-181)."""
    x = np.asarray(x, dtype=float)
    sd = _outer_signed(dom.outer, x)
    for h in dom.holes:
        sd = min(sd, _norm(x - h.center) - h.radius)
    if hasattr(dom.outer, "notch"):
        sd = min(sd, notch_signed(dom.outer.notch, x))
    return sd


# ---------------------------------------------------------------------------
# anchor generators


def circle_points(center, radius: float, m: int, component: int = -1,
                  phase: float = 0.0) -> BoundaryPointSet:
    """m points at angles 2*pi*(k + phase)/m (S/geometry.py:250-258 at phase 0)."""
    if m < 1:
        raise ValidationError("point count must be >= 1")
    center = np.asarray(center, dtype=float)
    ang = 2.0 * np.pi * (np.arange(m) + phase) / m
    pts = np.stack([center[0] + radius * np.cos(ang), center[1] + radius * np.sin(ang)], axis=1)
    block = AnchorBlock("circle", 0, m, component, center, radius, True, float(phase))
    return BoundaryPointSet(pts, np.full(m, component), ang, (block,))


def square_arc_to_point(h: float, s: float) -> np.ndarray:
    """Arc length s in [0, 8h) -> point on [-h,h]^2, start (h,-h), ccw
    (S/geometry.py:276-285)."""
    s = s % (8.0 * h)
    if s < 2.0 * h:
        return np.array([h, -h + s])
    if s < 4.0 * h:
        return np.array([h - (s - 2.0 * h), h])
    if s < 6.0 * h:
        return np.array([-h, h - (s - 4.0 * h)])
    return np.array([-h + (s - 6.0 * h), -h])


def square_points(center, halfwidth: float, m: int, component: int = -1,
                  phase: float = 0.0) -> BoundaryPointSet:
    """m points at arc length 8h*(k + phase)/m ccw from the bottom-right
    corner (S/geometry.py:261-273 at phase 0)."""
    if m < 1:
        raise ValidationError("point count must be >= 1")
    center = np.asarray(center, dtype=float)
    h = halfwidth
    s = (8.0 * h) * (np.arange(m) + phase) / m
    pts = np.stack([center + square_arc_to_point(h, si) for si in s])
    block = AnchorBlock("square", 0, m, component, center, h, True, float(phase))
    return BoundaryPointSet(pts, np.full(m, component), s, (block,))


def fibonacci_hemisphere(n: int, sign: float = 1.0) -> np.ndarray:
    """n Fibonacci-lattice points on the unit hemisphere sign*z > 0:
    z_k = sign*(k + 1/2)/n, azimuth k * golden angle (BASELINE cfg4)."""
    k = np.arange(n, dtype=float)
    z = (k + 0.5) / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = k * (np.pi * (3.0 - math.sqrt(5.0)))
    return np.stack([r * np.cos(phi), r * np.sin(phi), sign * z], axis=1)


def fibonacci_sphere(n: int, radius: float = 1.0) -> np.ndarray:
    """n Fibonacci-lattice points on the sphere of the given radius."""
    k = np.arange(n, dtype=float)
    z = 1.0 - (2.0 * k + 1.0) / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = k * (np.pi * (3.0 - math.sqrt(5.0)))
    return radius * np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def generic_points(points, component: int = -1) -> BoundaryPointSet:
    """An unstructured anchor family (empty blocks => generic packing)."""
    pts = np.ascontiguousarray(points, dtype=float)
    m = pts.shape[0]
    return BoundaryPointSet(pts, np.full(m, component), np.arange(m, dtype=float), ())


def concat_point_sets(sets) -> BoundaryPointSet:
    pts = np.concatenate([s.points for s in sets], axis=0)
    ids = np.concatenate([s.component_ids for s in sets])
    par = np.concatenate([s.params for s in sets])
    blocks = []
    off = 0
    for s in sets:
        for b in s.blocks:
            blocks.append(replace(b, start=b.start + off))
        off += len(s)
    return BoundaryPointSet(pts, ids, par, tuple(blocks))
