"""Closed-form checks of the production FP32 samplers on the GPU (north_star:
"where the Poisson kernel is known in closed form (disk, ball), entries also
match it within 4 binomial standard errors").

1. The samplers themselves, one step at a time (em_debug_step -> the same
   device functions the walk kernel runs: tangent_step, tangent_step3,
   roll_step2, roll_step3, and the woe / max steps).  From a start point x,
   every landing point of a walk-on-spheres step lies on ONE sphere in
   whitened coordinates w = K^{-1/2} x, and is distributed by that ball's
   harmonic measure seen from the start point -- the disk / ball Poisson
   kernel, whose law has a closed-form CDF (2D: the exit angle about the
   centre; 3D: the cosine of the polar angle, plus a uniform azimuth).  The
   sphere is FITTED to the CUDA landing points (least squares, no kernel
   formula reused), then checked: all points on it, the start point inside
   it, the whole ball inside the domain, and the law against the closed form
   by Kolmogorov-Smirnov over 2e6 samples per start point (>= 1e7 per
   sampler).  Start points: the BASELINE configs' own poles plus points
   close to the boundary, on every production chain (cfg2 tangent balls in
   the whitened parallelogram, cfg3 rolling / hole-tangent disks in the
   annulus, cfg4 rolling balls, cfg5 tangent balls with the notch planes),
   and the max / woe chains.

2. Whole walks against the Poisson kernel of the unit disk / ball with K = I.
   EM_FLAG_TANGENT_ON_IDENTITY runs the rolling chains on K = I, where the
   rolling ball IS the domain (shrunk by 1e-6): its first step samples the
   domain's exit law exactly.  cfg1's 128 arcs (32 poles x 1e6 walks) and
   the unit ball with cfg4's 2048 mirrored Fibonacci cells (64 poles x 1e6
   walks, every chain incl. the bit-exact REF64 mirror) against the
   cell-integrated Poisson kernel, with SURVEY Appendix B's three statistics:
   max |z| against the Bonferroni threshold, the number of |z| > 4 against
   the binomial 99.9% quantile, per-row chi^2 p-values (KS-uniform); plus a
   KS test of >= 1e7 exit angles / polar cosines against the closed-form
   CDF.  The eps-shell bias (eps = 1e-5 .. 1e-4, a relative shift of the
   exit law of order eps) is far below one standard error at these sizes
   ("after removing the eps-shell bias": it is removed by bounding it).
"""

import math

import numpy as np
import pytest

from helpers import bonferroni_z, exceed_quantile, poisson_cell_probs_disk

pytestmark = pytest.mark.gpu

KS_LEVEL = 1e-4  # per KS test (fixed seeds: deterministic per build)


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import _native, backend

    _native.require_device(0)
    return backend


# ---------------------------------------------------------------------------
# closed-form laws


def disk_angle_cdf(phi, rho, d):
    """Exit angle phi in (-pi, pi] about the centre, measured from the start
    point's direction, of Brownian motion from distance d in a disk of radius
    rho: 1/2 + atan((rho + d)/(rho - d) tan(phi / 2)) / pi."""
    return 0.5 + np.arctan((rho + d) / (rho - d) * np.tan(phi / 2.0)) / np.pi


def ball_cos_cdf(t, rho, d):
    """CDF of t = cos(polar angle from the start point's direction) of the
    exit point of a ball of radius rho from distance d (3D Poisson kernel)."""
    t = np.clip(t, -1.0, 1.0)
    if d < 1e-4 * rho:  # centred ball (d is fit noise): uniform
        return (t + 1.0) / 2.0
    s = np.sqrt(rho * rho + d * d - 2.0 * rho * d * t)
    return (rho * rho - d * d) / (2.0 * d) * (1.0 / s - 1.0 / (rho + d))


def fit_sphere(w):
    """Least-squares sphere through points w (n, d): |w|^2 = 2 c.w + k."""
    a = np.column_stack([2.0 * w, np.ones(len(w))])
    b = np.einsum("ij,ij->i", w, w)
    sol, *_ = np.linalg.lstsq(a, b, rcond=None)
    c = sol[:-1]
    rho = math.sqrt(sol[-1] + c @ c)
    return c, rho


def ks_p(sample, cdf):
    from scipy import stats

    return float(stats.kstest(sample, cdf).pvalue)


# ---------------------------------------------------------------------------
# 1. the samplers, one step at a time


def _start_points(cfg, rng):
    """Two of the config's poles and two points close to the boundary (found
    by moving a pole towards its nearest boundary point)."""
    from paper_2409_03686_b200.geometry import dist_to_boundary

    idx = [0, cfg.n_poles // 2 + 3]
    pts = [cfg.poles[i] for i in idx]
    for i, frac in ((1, 0.97), (cfg.n_poles // 3, 0.995)):
        p = cfg.poles[i]
        # nearest boundary direction by sampling: the point p + t u that
        # shrinks the distance fastest
        best = None
        for u in rng.normal(size=(400, cfg.d)):
            u /= np.linalg.norm(u)
            t = dist_to_boundary(cfg.dom, p)
            q = p + 0.98 * t * u
            if best is None or dist_to_boundary(cfg.dom, q) < best[0]:
                best = (dist_to_boundary(cfg.dom, q), u, t)
        _, u, t = best
        pts.append(p + frac * t * u)
    return np.array(pts)


def _check_one_step(B, cfg, plan, start, n, rng, label):
    from paper_2409_03686_b200.geometry import dist_to_boundary

    a = cfg.kt.k_sqrt
    ainv = np.linalg.inv(a)
    x = np.repeat(start[None, :], n, axis=0)
    words = rng.integers(0, 2**32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    y, mask = plan.debug_step(x, words)
    assert np.all(mask == 1.0), (label, "interior start point must walk")
    w = y @ ainv.T  # whitened landing points (x = A w, A symmetric)
    z = ainv @ start
    c, rho = fit_sphere(w)
    r = np.linalg.norm(w - c, axis=1)
    # every landing point on the one fitted sphere (FP32 coordinates)
    assert np.max(np.abs(r - rho)) <= 2e-5 + 2e-5 * rho, (label, np.max(np.abs(r - rho)), rho)
    d = float(np.linalg.norm(z - c))
    assert d < rho * (1 - 1e-7), (label, "start point outside its ball", d, rho)
    # the whole ball inside the domain (sampled on its surface, world units)
    u = rng.normal(size=(2000, cfg.d))
    u /= np.linalg.norm(u, axis=1)[:, None]
    sd = np.array([dist_to_boundary(cfg.dom, a @ (c + rho * v)) for v in u])
    assert sd.min() >= -1e-6, (label, "ball leaves the domain", sd.min())
    # the law: harmonic measure of the ball seen from z
    if cfg.d == 2:
        if d < 1e-4 * rho:  # centred ball (d is fit noise): uniform angle
            phi = np.arctan2(w[:, 1] - c[1], w[:, 0] - c[0])
            p = ks_p(phi, lambda t: (t + np.pi) / (2 * np.pi))
        else:
            e = (z - c) / d
            v = (w - c) / rho
            phi = np.arctan2(e[0] * v[:, 1] - e[1] * v[:, 0], v @ e)
            p = ks_p(phi, lambda t: disk_angle_cdf(t, rho, d))
        assert p > KS_LEVEL, (label, "exit law", p, d / rho)
        return rho, d
    v = (w - c) / np.linalg.norm(w - c, axis=1)[:, None]
    e = (z - c) / d if d >= 1e-4 * rho else np.array([0.0, 0.0, 1.0])
    t = v @ e
    p1 = ks_p(t, lambda s: ball_cos_cdf(s, rho, d))
    # azimuth about e: uniform
    f1 = np.cross(e, [1.0, 0.0, 0.0] if abs(e[0]) < 0.9 else [0.0, 1.0, 0.0])
    f1 /= np.linalg.norm(f1)
    f2 = np.cross(e, f1)
    az = np.arctan2(v @ f2, v @ f1)
    p2 = ks_p(az, lambda s: (s + np.pi) / (2 * np.pi))
    assert p1 > KS_LEVEL and p2 > KS_LEVEL, (label, "exit law", p1, p2, d / rho)
    return rho, d


@pytest.mark.parametrize("idx,chain", [(2, "tangent"), (3, "tangent"), (4, "tangent"),
                                       (5, "tangent"), (2, "max"), (3, "max"), (4, "max"),
                                       (5, "max"), (2, "woe"), (4, "woe")])
def test_sampler_one_step_is_a_ball_harmonic_measure(B, idx, chain):
    """One step of each production sampler from interior and near-boundary
    points: landing points on one whitened sphere inside the domain, with
    the closed-form disk / ball Poisson-kernel law (KS, 2e6 samples per
    start point)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx)
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    rng = np.random.default_rng(1000 + 10 * idx + len(chain))
    starts = _start_points(cfg, rng)
    with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles[:1], cfg.eps, 10**6, s0, s1, precision="fp32",
                chain=chain) as plan:
        assert plan.chain == chain
        seen = []
        for j, st in enumerate(starts):
            seen.append(_check_one_step(B, cfg, plan, st, 2_000_000, rng,
                                        f"cfg{idx}/{chain}/start{j}"))
    if chain in ("woe", "max"):  # walk on spheres CENTRED at the point
        assert max(d / rho for rho, d in seen) < 1e-4, seen
    if chain == "tangent":
        # the tangent / rolling chains take OFF-centre balls near the
        # boundary (that is what makes them fast): some start point sits
        # well away from its ball's centre
        assert max(d / rho for rho, d in seen) > 0.3, seen


# ---------------------------------------------------------------------------
# 2. whole walks on K = I: the rolling ball is the domain


def test_rolling_disk_on_identity_is_the_disk_poisson_kernel(B):
    """roll_step2 on the unit disk with K = I: exit angles of 1.2e7 walks
    from three poles follow the closed-form Poisson-kernel CDF (KS), almost
    every walk ends after its first step, and cfg1's 32 poles x 1e6 walks
    match the cell-integrated kernel of the 128 arcs (Appendix B)."""
    from paper_2409_03686_b200 import _native, configs

    cfg = configs.get(1)
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 2, cfg.eps)
    flags = _native.EM_FLAG_TANGENT_ON_IDENTITY
    starts = np.array([[0.5, 0.0], [-0.9 * 0.6, 0.9 * 0.8], [0.05, -0.1]])
    with B.Plan(geom, cfg.kt.k_sqrt, starts, cfg.eps, 10**6, s0, s1, precision="fp32",
                chain="tangent", flags=flags) as plan:
        assert plan.chain == "tangent"
        x, steps, _ = plan.exits(77, 4_000_000)
    assert np.mean(steps == 1) > 0.999, np.mean(steps == 1)
    for i, p in enumerate(starts):
        xi = x[i * 4_000_000:(i + 1) * 4_000_000]
        r = float(np.linalg.norm(p))
        rel = np.arctan2(xi[:, 1], xi[:, 0]) - math.atan2(p[1], p[0])
        rel = np.mod(rel + np.pi, 2 * np.pi) - np.pi
        pv = ks_p(rel, lambda t: disk_angle_cdf(t, 1.0, r))
        assert pv > KS_LEVEL, (i, pv)
    # counts in cfg1's arcs vs the cell-integrated kernel
    n = 10**6
    with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, precision="fp32",
                chain="tangent", flags=flags) as plan:
        res = plan.run(cfg.seed, n)
    assert np.array_equal(res.counts.sum(1), np.full(cfg.n_poles, n))
    probs = np.array([poisson_cell_probs_disk(p, 128) for p in cfg.poles])
    _appendix_b_one_sample(res.raw1, probs, n, "cfg1 rolling")


def _appendix_b_one_sample(counts, probs, n, label):
    """SURVEY Appendix B against known cell probabilities: Bonferroni max |z|,
    |z|>4 exceedances within the binomial 99.9% quantile, per-row chi^2
    goodness-of-fit p-values KS-uniform (and none below 1e-4 / rows)."""
    from scipy import stats

    counts = np.asarray(counts, float)
    z = (counts / n - probs) / np.sqrt(probs * (1 - probs) / n)
    m = z.size
    assert np.abs(z).max() <= bonferroni_z(m), (label, np.abs(z).max(), bonferroni_z(m))
    assert int((np.abs(z) > 4).sum()) <= exceed_quantile(m), (label, int((np.abs(z) > 4).sum()))
    pr = []
    for c, p in zip(counts, probs):
        e = p / p.sum() * n
        pr.append(stats.chi2.sf(float(np.sum((c - e) ** 2 / e)), len(c) - 1))
    pr = np.array(pr)
    assert pr.min() > 1e-4 / len(pr), (label, pr.min())
    assert stats.kstest(pr, "uniform").pvalue > 1e-4, (label, "row p-values not uniform")


@pytest.fixture(scope="module")
def ball_cells():
    """Cell-integrated 3D Poisson kernel of the unit ball over cfg4's 2048
    mirrored Fibonacci Voronoi cells: midpoint quadrature on a 2^22-point
    Fibonacci sphere (equal-area points), each point binned to its nearest
    anchor.  Returns (anchors, quadrature points, their cell ids)."""
    from scipy.spatial import cKDTree

    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.geometry import fibonacci_sphere

    anchors = configs.get(4).fam1.points
    q = fibonacci_sphere(1 << 22, 1.0)
    _, cell = cKDTree(anchors).query(q)
    return anchors, q, cell


def _ball_probs(poles, q, cell, n_cells):
    out = np.empty((len(poles), n_cells))
    w = 1.0 / len(q)  # (4 pi / Nq) x (1 / 4 pi)
    for i, p in enumerate(poles):
        r2 = float(p @ p)
        dist3 = np.sum((q - p) ** 2, axis=1) ** 1.5
        out[i] = np.bincount(cell, weights=(1.0 - r2) / dist3 * w, minlength=n_cells)
    return out


@pytest.mark.parametrize("precision,chain", [("fp32", "tangent"), ("fp32", "max"),
                                             ("fp32", "woe"), ("ref64", "woe")])
def test_unit_ball_cfg4_cells_match_3d_poisson_kernel(B, ball_cells, precision, chain):
    """Unit ball, K = I, cfg4's 2048 mirrored Fibonacci cells, 64 of cfg4's
    poles (r = 0.6) x 1e6 walks, every chain (tangent = rolling balls forced
    on K = I, i.e. the ball itself): entries against the cell-integrated 3D
    Poisson kernel (1 - |z|^2) / (4 pi |z - y|^3) with Appendix B's three
    statistics."""
    from paper_2409_03686_b200 import _native, configs
    from paper_2409_03686_b200.conductivity import make_tensor
    from paper_2409_03686_b200.geometry import Ball, Domain

    anchors, q, cell = ball_cells
    cfg = configs.get(4).subset(64)
    dom = Domain(3, Ball(np.zeros(3), 1.0), (), frozenset())
    geom = B.pack_geometry(dom)
    s0 = B.pack_side(None, 3, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 3, cfg.eps)
    ident = make_tensor(np.eye(3)).k_sqrt
    flags = _native.EM_FLAG_TANGENT_ON_IDENTITY if chain == "tangent" else 0
    n = 10**6
    with B.Plan(geom, ident, cfg.poles, cfg.eps, 10**6, s0, s1, precision=precision,
                chain=chain, flags=flags) as plan:
        assert plan.chain == chain
        res = plan.run(cfg.seed, n)
    assert np.array_equal(res.counts.sum(1), np.full(cfg.n_poles, n))
    probs = _ball_probs(cfg.poles, q, cell, len(anchors))
    assert np.allclose(probs.sum(1), 1.0, atol=2e-3)
    probs /= probs.sum(1, keepdims=True)
    _appendix_b_one_sample(res.raw1, probs, n, f"ball/{precision}/{chain}")


def test_rolling_ball_on_identity_is_the_ball_poisson_kernel(B):
    """roll_step3 on the unit ball with K = I: 1.2e7 exits from three poles,
    polar cosine about the pole direction against the closed-form CDF and a
    uniform azimuth (KS); almost every walk ends after one step."""
    from paper_2409_03686_b200 import _native, configs
    from paper_2409_03686_b200.conductivity import make_tensor
    from paper_2409_03686_b200.geometry import Ball, Domain

    cfg = configs.get(4)
    dom = Domain(3, Ball(np.zeros(3), 1.0), (), frozenset())
    geom = B.pack_geometry(dom)
    s0 = B.pack_side(None, 3, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 3, cfg.eps)
    starts = np.array([[0.0, 0.0, 0.6], [0.5, -0.5, 0.5], [0.02, 0.03, -0.05]])
    with B.Plan(geom, make_tensor(np.eye(3)).k_sqrt, starts, cfg.eps, 10**6, s0, s1,
                precision="fp32", chain="tangent",
                flags=_native.EM_FLAG_TANGENT_ON_IDENTITY) as plan:
        x, steps, _ = plan.exits(99, 4_000_000)
    assert np.mean(steps == 1) > 0.999, np.mean(steps == 1)
    for i, p in enumerate(starts):
        xi = x[i * 4_000_000:(i + 1) * 4_000_000]
        v = xi / np.linalg.norm(xi, axis=1)[:, None]
        r = float(np.linalg.norm(p))
        e = p / r
        p1 = ks_p(v @ e, lambda s: ball_cos_cdf(s, 1.0, r))
        f1 = np.cross(e, [1.0, 0.0, 0.0] if abs(e[0]) < 0.9 else [0.0, 1.0, 0.0])
        f1 /= np.linalg.norm(f1)
        f2 = np.cross(e, f1)
        p2 = ks_p(np.arctan2(v @ f2, v @ f1), lambda s: (s + np.pi) / (2 * np.pi))
        assert p1 > KS_LEVEL and p2 > KS_LEVEL, (i, p1, p2)


def test_annulus_rolling_chain_hit_probability_on_identity(B):
    """roll_step2 with the concentric hole (cfg3's chain) on K = I: the
    inner-circle hit probability ln(R/r)/ln(R/rho) (T/test_walk.py:70-78)
    at 4e6 walks per start radius, exact binomial test."""
    from scipy.stats import binomtest

    from paper_2409_03686_b200 import _native, configs
    from paper_2409_03686_b200.conductivity import make_tensor

    cfg = configs.get(3)
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 2, cfg.eps)
    starts = np.array([[0.95, 0.0], [0.0, 0.7], [-0.55, 0.05]])
    n = 4_000_000
    with B.Plan(geom, make_tensor(np.eye(2)).k_sqrt, starts, cfg.eps, 10**6, s0, s1,
                precision="fp32", chain="tangent",
                flags=_native.EM_FLAG_TANGENT_ON_IDENTITY) as plan:
        assert plan.chain == "tangent"
        res = plan.run(5, n)
    hit = res.counts[:, s0.size:].sum(1)
    for i, p in enumerate(starts):
        r = float(np.linalg.norm(p))
        prob = math.log(1.0 / r) / math.log(1.0 / 0.5)
        pv = binomtest(int(hit[i]), n, prob).pvalue
        assert pv > 1e-4 / len(starts), (r, hit[i] / n, prob, pv)
