"""Cell measures sigma of Voronoi weight families by boundary quadrature on
the GPU.

The reference computes sigma(omega_j) exactly for uniform circle blocks and by
dense midpoint sampling of the anchor blocks' shapes otherwise, and rejects
unstructured ("generic") anchors (S/weights.py:155-181, 36-44 with S/ =
/root/reference/pkg/src/exitmeasure/) -- exactly the BASELINE cfg4
(Fibonacci cells) and cfg5 (L-box squares) families.  Here the boundary of
the DOMAIN is sampled with equal-weight midpoint quadrature (circles by
angle, spheres by the equal-area (z, theta) product grid the reference uses,
box / L-box faces by square grids) and every sample is binned on the GPU with
the walk kernel's rule -- owner component -> side -> nearest anchor -- so
sigma is the measure of each anchor's cell as the estimator actually bins.
"""

from __future__ import annotations

import math

import numpy as np

from .backend import Plan, pack_geometry, pack_side
from .errors import ValidationError


def _circle(center, radius, q):
    ang = 2.0 * np.pi * (np.arange(q) + 0.5) / q
    pts = np.stack([center[0] + radius * np.cos(ang), center[1] + radius * np.sin(ang)], axis=1)
    return pts, np.full(q, 2.0 * np.pi * radius / q)


def _sphere(center, radius, q):
    qz = max(int(math.ceil(math.sqrt(q / 2.0))), 4)
    qz += qz % 2  # even: no sample ring on the equator (a tie between hemispheres)
    qt = 2 * qz
    z = -radius + 2.0 * radius * (np.arange(qz) + 0.5) / qz
    th = 2.0 * np.pi * (np.arange(qt) + 0.5) / qt
    zz, tt = np.meshgrid(z, th, indexing="ij")
    rho = np.sqrt(np.maximum(radius**2 - zz**2, 0.0))
    pts = np.stack([center[0] + rho * np.cos(tt), center[1] + rho * np.sin(tt), center[2] + zz],
                   axis=-1).reshape(-1, 3)
    return pts, np.full(pts.shape[0], 4.0 * np.pi * radius**2 / pts.shape[0])


def _rect_face(axis, value, lo, hi, h):
    """Midpoint grid of spacing ~h on the face {x_axis = value} over the
    box [lo, hi] in the other two axes (3D)."""
    o = [a for a in range(3) if a != axis]
    nu = max(1, int(round((hi[0] - lo[0]) / h)))
    nv = max(1, int(round((hi[1] - lo[1]) / h)))
    u = lo[0] + (np.arange(nu) + 0.5) * (hi[0] - lo[0]) / nu
    v = lo[1] + (np.arange(nv) + 0.5) * (hi[1] - lo[1]) / nv
    uu, vv = np.meshgrid(u, v, indexing="ij")
    pts = np.empty((uu.size, 3))
    pts[:, axis] = value
    pts[:, o[0]] = uu.ravel()
    pts[:, o[1]] = vv.ravel()
    w = (hi[0] - lo[0]) * (hi[1] - lo[1]) / uu.size
    return pts, np.full(uu.size, w)


def boundary_samples(dom, spacing: float):
    """Equal-weight midpoint quadrature of the whole boundary of ``dom`` with
    roughly the given sample spacing: (points, weights)."""
    d = dom.dimension
    parts = []
    outer = dom.outer
    if hasattr(outer, "radius"):
        c = np.asarray(outer.center, float)
        r = float(outer.radius)
        if d == 2:
            parts.append(_circle(c, r, max(64, int(2 * np.pi * r / spacing))))
        else:
            parts.append(_sphere(c, r, max(256, int(4 * np.pi * r * r / spacing**2))))
    else:
        c = np.asarray(outer.center, float)
        h = float(outer.halfwidth)
        lo, hi = c - h, c + h
        if d == 2:
            n = max(4, int(2 * h / spacing))
            t = lo[0] + (np.arange(n) + 0.5) * (2 * h) / n
            s = lo[1] + (np.arange(n) + 0.5) * (2 * h) / n
            w = np.full(n, 2 * h / n)
            for pts in (np.stack([np.full(n, hi[0]), s], 1), np.stack([t, np.full(n, hi[1])], 1),
                        np.stack([np.full(n, lo[0]), s], 1), np.stack([t, np.full(n, lo[1])], 1)):
                parts.append((pts, w))
        else:
            notch = getattr(outer, "notch", None)
            for axis in range(3):
                o = [a for a in range(3) if a != axis]
                for val in (lo[axis], hi[axis]):
                    pts, w = _rect_face(axis, val, lo[o], hi[o], spacing)
                    if notch is not None:
                        keep = ~((pts[:, 0] > notch[0]) & (pts[:, 1] > notch[1]))
                        if axis == 0 and val == hi[0]:
                            keep = pts[:, 1] < notch[1]
                        if axis == 1 and val == hi[1]:
                            keep = pts[:, 0] < notch[0]
                        pts, w = pts[keep], w[keep]
                    parts.append((pts, w))
            if notch is not None:
                nx, ny = notch
                parts.append(_rect_face(0, nx, np.array([ny, lo[2]]), np.array([hi[1], hi[2]]),
                                        spacing))
                parts.append(_rect_face(1, ny, np.array([nx, lo[2]]), np.array([hi[0], hi[2]]),
                                        spacing))
    for hole in dom.holes:
        c = np.asarray(hole.center, float)
        r = float(hole.radius)
        if d == 2:
            parts.append(_circle(c, r, max(64, int(2 * np.pi * r / spacing))))
        else:
            parts.append(_sphere(c, r, max(256, int(4 * np.pi * r * r / spacing**2))))
    pts = np.concatenate([p for p, _ in parts])
    w = np.concatenate([w for _, w in parts])
    return pts, w


def cell_measures(dom, fam0, fam1, eps: float = 1e-6, samples_per_anchor: int = 100,
                  precision: str = "ref64", device: int | None = None,
                  spacing: float | None = None):
    """(sigma0, sigma1): boundary measure of each anchor's cell under the
    estimator's binning rule, by GPU-binned midpoint quadrature with about
    ``samples_per_anchor`` samples per anchor (or an explicit sample
    ``spacing``, e.g. one that nests in square bins for exact areas)."""
    d = dom.dimension
    s0 = pack_side(fam0, d, eps)
    s1 = pack_side(fam1, d, eps)
    n_anchors = s0.size + s1.size
    if n_anchors == 0:
        raise ValidationError("no anchors")
    if spacing is None:
        total = float(boundary_samples(dom, 0.05)[1].sum())  # boundary measure
        if d == 2:
            spacing = total / (samples_per_anchor * n_anchors)
        else:
            spacing = math.sqrt(total / (samples_per_anchor * n_anchors))
    pts, w = boundary_samples(dom, spacing)
    centre = np.asarray(dom.outer.center, float)
    if hasattr(dom.outer, "notch"):
        centre = np.asarray(dom.outer.center, float) - 0.5 * dom.outer.halfwidth
    geom = pack_geometry(dom)
    with Plan(geom, np.eye(d), centre[None, :], eps, 1, s0, s1, precision=precision,
              device=device) as plan:
        comp, side, bins = plan.bin_points(pts)
    sig0 = np.bincount(bins[side == 0], weights=w[side == 0], minlength=s0.size)[: s0.size]
    sig1 = np.bincount(bins[side == 1], weights=w[side == 1], minlength=s1.size)[: s1.size]
    return sig0, sig1
