"""The exit-point samplers of the FP32 tangent / rolling-ball chains
(csrc/walk_f32.cu: tangent_step, tangent_step3, roll_step2, roll_step3),
restated in float64 numpy and checked against the harmonic measure they
claim to sample: the Poisson kernel of a disk / ball seen from an interior
point.  CPU only -- the GPU suite checks the kernels themselves against the
oracle (test_gpu_parity.py) and tools/soak_tangent.py at scale."""

import numpy as np
from scipy import stats


def _disk_exit(rho, m, psi):
    """2D: point at depth m below the near point of a disk of radius rho
    (distance d = rho - m from the centre); Moebius image of psi uniform in
    (-pi/2, pi/2): depth below the tangent line and tangential offset."""
    N = m * np.sin(psi)
    D = (2 * rho - m) * np.cos(psi)
    g = 2 * rho / (N * N + D * D)
    return g * N * N, g * N * D


def _ball_exit_depth(rho, m, v2):
    """3D: depth below the near point, V2 = 2V uniform in (0, 2)."""
    d = rho - m
    g = m / (m + d * v2)
    return g * g * (2 - v2) * (rho + 0.5 * d * v2)


def test_disk_exit_lies_on_the_circle():
    rng = np.random.default_rng(1)
    rho = rng.uniform(0.1, 2.0, 10000)
    m = rho * rng.uniform(1e-6, 1.0, 10000)
    psi = rng.uniform(-np.pi / 2, np.pi / 2, 10000)
    dep, off = _disk_exit(rho, m, psi)
    # on the circle of radius rho centred rho below the tangent point
    assert np.allclose(off ** 2 + (rho - dep) ** 2, rho ** 2, rtol=1e-12, atol=1e-14)


def test_disk_exit_law_is_the_poisson_kernel():
    """Exit angle t (from the near point, about the centre) of the Moebius
    sample against the disk's Poisson kernel P(t) = (r^2 - d^2) / (2 pi
    (r^2 + d^2 - 2 r d cos t)) seen from distance d on the near axis."""
    rng = np.random.default_rng(2)
    for rho, m in ((1.0, 0.3), (1.0, 1.0), (0.5, 1e-3), (2.0, 1.7)):
        psi = rng.uniform(-np.pi / 2, np.pi / 2, 200000)
        dep, off = _disk_exit(rho, m, psi)
        t = np.arctan2(off, rho - dep)
        d = rho - m
        grid = np.linspace(-np.pi, np.pi, 20001)
        pdf = (rho ** 2 - d ** 2) / (2 * np.pi * (rho ** 2 + d ** 2 - 2 * rho * d * np.cos(grid)))
        cdf = np.concatenate([[0], np.cumsum(0.5 * (pdf[1:] + pdf[:-1]) * np.diff(grid))])
        cdf /= cdf[-1]
        p = stats.kstest(t, lambda x: np.interp(x, grid, cdf)).pvalue
        assert p > 1e-4, (rho, m, p)


def test_ball_exit_law_is_the_poisson_kernel():
    """3D: the depth formula's law of cos(theta) = 1 - dep / rho against the
    ball's Poisson kernel, whose law in u = cos(theta) has CDF
    F(u) = (r^2 - d^2) / (2 d) (1 / s(u) - 1 / (r + d)), s(u) = |z - y| =
    sqrt(r^2 + d^2 - 2 r d u); the azimuth is uniform by symmetry."""
    rng = np.random.default_rng(3)
    for rho, m in ((1.0, 0.25), (1.0, 1.0), (0.4, 1e-3), (2.0, 1.9)):
        # 16-bit V as in the kernel: V2 = (2k + 1) / 2^16
        k = rng.integers(0, 1 << 16, 200000)
        v2 = (2 * k + 1) / 65536.0
        dep = _ball_exit_depth(rho, m, v2)
        assert (dep >= 0).all() and (dep <= 2 * rho * (1 + 1e-12)).all()
        u = 1 - dep / rho
        d = rho - m
        if d == 0:
            cdf = lambda x: (np.clip(x, -1, 1) + 1) / 2  # noqa: E731  (uniform)
        else:
            def cdf(x):
                x = np.clip(x, -1, 1)
                s = np.sqrt(rho ** 2 + d ** 2 - 2 * rho * d * x)
                return (rho ** 2 - d ** 2) / (2 * d) * (1 / s - 1 / (rho + d))
        p = stats.kstest(u, cdf).pvalue
        assert p > 1e-4, (rho, m, p)


def test_rolling_offset_and_near_side():
    """The rolling-ball centre offset in the rotated frame, w = x (al / a +
    be a) with al = 1 - R / |x|, be = rho_b / |Ax|, equals z - c for the ball
    of radius rho_b internally tangent at the radial projection p = R x /
    |x| (whitened z = x / a, inward normal -a x / |Ax|), and the near-side
    test al |x|^2 + be |Ax|^2 > 0 is (z - c) . n < 0."""
    rng = np.random.default_rng(4)
    a = np.array([0.5, np.sqrt(0.5), 1.0])
    R, rho_b = 1.0, 1.0 * a.min() / a.max() ** 2
    for _ in range(1000):
        x = rng.normal(size=3)
        x *= rng.uniform(0.05, 0.999) / np.linalg.norm(x)
        z = x / a
        p = z * R / np.linalg.norm(x)
        n = -(a * x) / np.linalg.norm(a * x)
        c = p + rho_b * n
        al = 1 - R / np.linalg.norm(x)
        be = rho_b / np.linalg.norm(a * x)
        w = x * (al / a + be * a)
        assert np.allclose(w, z - c, atol=1e-12)
        assert (al * (x @ x) + be * ((a * x) @ (a * x)) > 0) == ((z - c) @ n < 0)


def test_rolling_radius_fits_the_ellipsoid():
    """rho_b = R min(a) / max(a)^2 is the smallest curvature radius of the
    whitened ellipsoid |diag(a) z| <= R: the rolling ball tangent at random
    boundary points stays inside (sampled on its surface)."""
    rng = np.random.default_rng(5)
    a = np.array([0.5, np.sqrt(0.5), 1.0])
    R = 1.0
    rho_b = R * a.min() / a.max() ** 2
    for _ in range(300):
        xb = rng.normal(size=3)
        xb *= R / np.linalg.norm(xb)  # boundary point, x-coordinates
        p = xb / a
        n = -(a * xb) / np.linalg.norm(a * xb)
        c = p + rho_b * (1 - 1e-9) * n
        u = rng.normal(size=(2000, 3))
        u /= np.linalg.norm(u, axis=1)[:, None]
        y = c + rho_b * (1 - 1e-9) * u
        assert (np.linalg.norm(y * a, axis=1) <= R * (1 + 1e-9)).all()


def test_annulus_disk_radii_clear_both_circles():
    """2D annulus (cfg3: K eigenvalues (1, 5) rotated, rho = 0.5, R = 1):
    disks of radius r = (R - rho) / (2 max a) tangent to the outer ellipse at
    a radial projection stay inside it (r <= the Blaschke radius) and off
    the hole; disks of that radius tangent to the hole from outside miss the
    hole and stay inside R (all in whitened coordinates, sampled on the disk
    boundary)."""
    rng = np.random.default_rng(6)
    a = np.array([1 / np.sqrt(5.0), 1.0])
    R, rho = 1.0, 0.5
    r = (R - rho) / (2 * a.max())
    assert r <= R * a.min() / a.max() ** 2
    th = np.linspace(0, 2 * np.pi, 721)
    ring = np.column_stack([np.cos(th), np.sin(th)])
    for _ in range(500):
        phi = rng.uniform(0, 2 * np.pi)
        xd = np.array([np.cos(phi), np.sin(phi)])
        for rad, sign in ((R, -1.0), (rho, 1.0)):  # outer: inward; hole: outward
            p = rad * xd / a
            n = sign * (a * rad * xd) / np.linalg.norm(a * rad * xd)
            c = p + r * (1 - 1e-9) * n
            y = c + r * (1 - 1e-9) * ring
            xr = np.linalg.norm(y * a, axis=1)
            assert (xr <= R * (1 + 1e-9)).all() and (xr >= rho * (1 - 1e-9)).all()
