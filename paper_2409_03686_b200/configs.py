"""The five BASELINE.json configurations as synthetic inputs.

Every config is fully synthetic (BASELINE.json names no dataset); seeds and
phases that BASELINE.json leaves open are fixed here and recorded in
DESIGN.md.  Each config yields the packed inputs of the exit-measure path:
domain, normalised K^{1/2}, poles, the two weight families (as structured
anchor blocks where the bins have closed form), the column split of the
result into A0 (accessible Gamma0) and A1 (inaccessible Gamma1) and, where
known in closed form, the Gamma1 cell measures sigma1.

Reference expressions: cfg1, cfg2 and cfg4 are a
gamma0=() domain with ONE anchor family whose columns are split into A0|A1
afterwards; cfg3 uses the reference's own annulus catalog entry; cfg5 (the
L-box) is not expressible in the reference and uses the notch extension.

cfg   domain / K                          poles   bins (G0+G1)   N/pole  eps
1     unit disk, K=I                      32      64+64 arcs     1e4     1e-4
2     unit square, K=[[2,.8],[.8,1]]      256     384+128 edges  1e5     1e-5
3     annulus .5<r<1, eig(1,5) rot pi/6   1024    512+512 arcs   1e6     1e-5
4     unit ball, R diag(1,2,4) R^T        1024    1024+1024 Fib  1e6     1e-5
5     L-box, [[3,1,0],[1,2,.5],[0,.5,1]]  4096    4050+4096 sq   1e6     1e-6
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .conductivity import ConductivityTensor, make_tensor
from .geometry import (Ball, Box, BoundaryPointSet, Domain, LBox, circle_points,
                       dist_to_boundary, fibonacci_hemisphere, fibonacci_sphere,
                       generic_points, square_points)

# fixed seeds (BASELINE.json leaves them open)
WALK_SEED = {1: 20240905, 2: 20240906, 3: 20240907, 4: 20240908, 5: 20240909}
CFG4_ROTATION_SEED = 2409
CFG5_POLE_SEED = 3686


@dataclass(eq=False)
class ExitConfig:
    index: int
    name: str
    dom: Domain
    kt: ConductivityTensor
    poles: np.ndarray
    eps: float
    n_rep: int  # walks per pole at full scale
    fam0: BoundaryPointSet | None
    fam1: BoundaryPointSet
    # how A0 / A1 are read off (raw0, raw1): (side, column indices)
    a0_cols: tuple
    a1_cols: tuple
    sigma1: np.ndarray | None
    seed: int
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def d(self) -> int:
        return self.dom.dimension

    @property
    def n_poles(self) -> int:
        return self.poles.shape[0]

    @property
    def total_walks(self) -> int:
        return self.n_poles * self.n_rep

    def split(self, raw0: np.ndarray, raw1: np.ndarray):
        """(A0, A1) column blocks of the raw count rows."""
        raws = (raw0, raw1)
        a0 = raws[self.a0_cols[0]][:, self.a0_cols[1]]
        a1 = raws[self.a1_cols[0]][:, self.a1_cols[1]]
        return a0, a1

    def subset(self, n_poles: int | None = None, n_rep: int | None = None) -> "ExitConfig":
        """A reduced copy: every k-th pole (so all angles/positions stay
        represented) and fewer walks per pole -- for parity tests and CPU
        baselines.  Pole order is preserved; pole indices are renumbered."""
        poles = self.poles
        if n_poles is not None and n_poles < poles.shape[0]:
            idx = np.linspace(0, poles.shape[0] - 1, n_poles).round().astype(int)
            poles = poles[idx]
        return ExitConfig(self.index, self.name, self.dom, self.kt, poles.copy(), self.eps,
                          int(n_rep or self.n_rep), self.fam0, self.fam1, self.a0_cols,
                          self.a1_cols, self.sigma1, self.seed, self.notes, dict(self.extra))


def _rot2(theta: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s], [s, c]])


def cfg1() -> ExitConfig:
    dom = Domain(2, Ball(np.zeros(2), 1.0), (), frozenset())
    # 128 arcs of 2pi/128 starting at angle 0: anchors at the arc midpoints
    fam1 = circle_points(np.zeros(2), 1.0, 128, component=0, phase=0.5)
    ang = 2.0 * np.pi * np.arange(32) / 32
    poles = 0.5 * np.stack([np.cos(ang), np.sin(ang)], axis=1)
    return ExitConfig(1, "cfg1_disk", dom, make_tensor(np.eye(2)), poles, 1e-4, 10**4, None,
                      fam1, (1, np.arange(0, 64)), (1, np.arange(64, 128)),
                      np.full(64, np.pi / 64), WALK_SEED[1],
                      "upper semicircle arcs 0..63 = Gamma0, lower 64..127 = Gamma1")


def cfg2() -> ExitConfig:
    dom = Domain(2, Box(np.array([0.5, 0.5]), 0.5), (), frozenset())
    # 512 edge-midpoint anchors ccw from the corner (1,0): right edge 0..127
    # (upward), top 128..255 (leftward), left 256..383, bottom 384..511
    fam1 = square_points(np.array([0.5, 0.5]), 0.5, 512, component=0, phase=0.5)
    g = np.arange(1, 17) / 17.0
    poles = np.array([[a, b] for a in g for b in g])
    a0 = np.concatenate([np.arange(0, 128), np.arange(256, 512)])
    return ExitConfig(2, "cfg2_square", dom, make_tensor([[2.0, 0.8], [0.8, 1.0]]), poles, 1e-5,
                      10**5, None, fam1, (1, a0), (1, np.arange(128, 256)),
                      np.full(128, 1.0 / 128), WALK_SEED[2],
                      "Gamma1 = top edge (anchors 128..255), Gamma0 = right+left+bottom")


def cfg3() -> ExitConfig:
    dom = Domain(2, Ball(np.zeros(2), 1.0), (Ball(np.zeros(2), 0.5),), frozenset({0}))
    rot = _rot2(np.pi / 6)
    k = rot @ np.diag([1.0, 5.0]) @ rot.T
    fam0 = circle_points(np.zeros(2), 1.0, 512, component=0)
    fam1 = circle_points(np.zeros(2), 0.5, 512, component=1)
    ang = 2.0 * np.pi * np.arange(512) / 512
    ring = np.stack([np.cos(ang), np.sin(ang)], axis=1)
    poles = np.concatenate([0.9 * ring, 0.7 * ring])
    return ExitConfig(3, "cfg3_annulus", dom, make_tensor(k), poles, 1e-5, 10**6, fam0, fam1,
                      (0, np.arange(512)), (1, np.arange(512)),
                      np.full(512, 2.0 * np.pi * 0.5 / 512), WALK_SEED[3],
                      "reference circle_points phase (cells centred at 2 pi k / 512)")


def cfg4_rotation() -> np.ndarray:
    q, _ = np.linalg.qr(np.random.default_rng(CFG4_ROTATION_SEED).normal(size=(3, 3)))
    return q


def cfg4() -> ExitConfig:
    dom = Domain(3, Ball(np.zeros(3), 1.0), (), frozenset())
    r = cfg4_rotation()
    k = r @ np.diag([1.0, 2.0, 4.0]) @ r.T
    k = 0.5 * (k + k.T)
    upper = fibonacci_hemisphere(1024, +1.0)
    lower = upper * np.array([1.0, 1.0, -1.0])  # exact mirror: side-first == global Voronoi
    fam1 = generic_points(np.concatenate([upper, lower]), component=0)
    poles = fibonacci_sphere(1024, 0.6)
    return ExitConfig(4, "cfg4_ball", dom, make_tensor(k), poles, 1e-5, 10**6, None, fam1,
                      (1, np.arange(1024)), (1, np.arange(1024, 2048)), None, WALK_SEED[4],
                      "mirrored Fibonacci hemisphere lattices z = +-(k+1/2)/1024")


def lbox_anchors():
    """Gamma0: 4050 squares of side 1/30 on the six outer faces of the
    L-box; Gamma1: 4096 squares of side 1/64 on the two notch faces."""
    def grid(u0, u1, v0, v1, h):
        nu = int(round((u1 - u0) / h))
        nv = int(round((v1 - v0) / h))
        u = u0 + (np.arange(nu) + 0.5) * h
        v = v0 + (np.arange(nv) + 0.5) * h
        uu, vv = np.meshgrid(u, v, indexing="ij")
        return uu.ravel(), vv.ravel()

    h0 = 1.0 / 30.0
    pts = []
    for z in (0.0, 1.0):  # bottom / top: the L-shape = three quadrants
        for (x0, x1, y0, y1) in ((0, .5, 0, .5), (.5, 1, 0, .5), (0, .5, .5, 1)):
            u, v = grid(x0, x1, y0, y1, h0)
            pts.append(np.stack([u, v, np.full_like(u, z)], axis=1))
    u, v = grid(0, 1, 0, 1, h0)  # x = 0: (y, z)
    pts.append(np.stack([np.zeros_like(u), u, v], axis=1))
    u, v = grid(0, 1, 0, 1, h0)  # y = 0: (x, z)
    pts.append(np.stack([u, np.zeros_like(u), v], axis=1))
    u, v = grid(0, .5, 0, 1, h0)  # x = 1: y in [0,.5]
    pts.append(np.stack([np.ones_like(u), u, v], axis=1))
    u, v = grid(0, .5, 0, 1, h0)  # y = 1: x in [0,.5]
    pts.append(np.stack([u, np.ones_like(u), v], axis=1))
    g0 = np.concatenate(pts)
    h1 = 1.0 / 64.0
    u, v = grid(.5, 1, 0, 1, h1)  # notch face x = .5: (y, z)
    f1 = np.stack([np.full_like(u, .5), u, v], axis=1)
    u, v = grid(.5, 1, 0, 1, h1)  # notch face y = .5: (x, z)
    f2 = np.stack([u, np.full_like(u, .5), v], axis=1)
    g1 = np.concatenate([f1, f2])
    return g0, g1


def cfg5_poles(n: int = 4096, dmin: float = 0.05, seed: int = CFG5_POLE_SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    dom = cfg5_domain()
    out = []
    while len(out) < n:
        p = rng.random(3)
        if dist_to_boundary(dom, p) > dmin:
            out.append(p)
    return np.asarray(out)


def cfg5_domain() -> Domain:
    return Domain(3, LBox(np.array([0.5, 0.5, 0.5]), 0.5, (0.5, 0.5)), (), frozenset({0}))


def cfg5() -> ExitConfig:
    dom = cfg5_domain()
    g0, g1 = lbox_anchors()
    k = np.array([[3.0, 1.0, 0.0], [1.0, 2.0, 0.5], [0.0, 0.5, 1.0]])
    return ExitConfig(5, "cfg5_lbox", dom, make_tensor(k), cfg5_poles(), 1e-6, 10**6,
                      generic_points(g0, 0), generic_points(g1, 1),
                      (0, np.arange(len(g0))), (1, np.arange(len(g1))),
                      np.full(len(g1), 1.0 / 4096), WALK_SEED[5],
                      "Gamma0 4050 squares of side 1/30 (4096 equal squares cannot tile area "
                      "4.5), Gamma1 2 x 32 x 64 squares of side 1/64")


CONFIGS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


def get(index: int) -> ExitConfig:
    return CONFIGS[int(index)]()
