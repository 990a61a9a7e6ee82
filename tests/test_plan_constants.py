"""Host unit tests of the FP32 kernel's closed-form plan constants
(csrc/plan_f32.cu, through em_f32_constant -- no device needed): every table
the tangent / rolling / sheared chains read is checked against its geometric
definition, recomputed here in float64 from the plan's geometry and K^{1/2}.
An error in these constants would otherwise surface only statistically."""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import backend
    from paper_2409_03686_b200.build_native import build, lib_path

    if not lib_path().exists():
        build()
    return backend


def _const(B, cfg, chain, name):
    geom = B.pack_geometry(cfg.dom)
    return B.f32_constant(geom, cfg.kt.k_sqrt, chain, cfg.eps, name).astype(np.float64)


def _normals(a):
    r = np.linalg.norm(a, axis=1)
    return r, a / r[:, None]


@pytest.mark.parametrize("idx", [5])
def test_tangent_face_tables_3d(B, idx):
    """t3: per nearest face i, cosines C_il = a_i . a_l of the unit whitened
    face normals, the tangent frame (e1 = unit part of a_{i+1} orthogonal to
    a_i, e2 = a_i x e1) components of every other normal, and the face-limit
    gains bt_l / (1 -+ C_il), 1 / (1 -+ C_il); tbt / tsb / tn the whitened
    half-widths, stop thresholds and notch planes."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx)
    a = cfg.kt.k_sqrt
    R, n = _normals(a)
    h = 0.5
    bt = h / R
    t3 = _const(B, cfg, "tangent", "t3").reshape(3, 24)
    assert np.allclose(_const(B, cfg, "tangent", "tbt"), bt, rtol=1e-6)
    assert np.allclose(_const(B, cfg, "tangent", "tsb"), bt - cfg.eps / R, rtol=1e-6, atol=1e-7)
    for i in range(3):
        j = (i + 1) % 3
        e1 = n[j] - (n[i] @ n[j]) * n[i]
        e1 /= np.linalg.norm(e1)
        e2 = np.cross(n[i], e1)
        T = t3[i]
        C, P1, P2 = T[0:3], T[3:6], T[6:9]
        Bm, tim, Bp, tip = T[9:12], T[12:15], T[15:18], T[18:21]
        for l in range(3):
            c = 1.0 if l == i else n[i] @ n[l]
            assert C[l] == pytest.approx(c, rel=1e-6, abs=1e-7)
            assert Bp[l] == pytest.approx(bt[l] / (1 + c), rel=1e-6)
            assert tip[l] == pytest.approx(1 / (1 + c), rel=1e-6)
            if l == i:
                assert Bm[l] > 1e37 and tim[l] == 0.0
                continue
            assert P1[l] == pytest.approx(n[l] @ e1, abs=1e-6)
            assert P2[l] == pytest.approx(n[l] @ e2, abs=1e-6)
            # a_l = C a_i + P1 e1 + P2 e2 is a unit vector
            assert C[l] ** 2 + P1[l] ** 2 + P2[l] ** 2 == pytest.approx(1.0, abs=2e-6)
            assert Bm[l] == pytest.approx(bt[l] / (1 - c), rel=1e-6)
            assert tim[l] == pytest.approx(1 / (1 - c), rel=1e-6)
        assert abs(P2[j]) < 1e-6 and P1[j] > 0  # e1 lies in the (a_i, a_j) plane
    notch = np.array([0.5, 0.5])
    frame = _const(B, cfg, "tangent", "frame")[:2]
    assert np.allclose(_const(B, cfg, "tangent", "tn"), (notch - frame) / R[:2], rtol=1e-6)


def test_tangent_parallelogram_2d(B):
    """cfg2: tcd = a_0 . a_1, tsd = sqrt(1 - tcd^2), tim / tip = 1 / (1 -+
    tcd), tbt = h / R_i, stored axes ax = R_i."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(2)
    R, n = _normals(cfg.kt.k_sqrt)
    c = n[0] @ n[1]
    assert _const(B, cfg, "tangent", "tcd")[0] == pytest.approx(c, rel=1e-6)
    assert _const(B, cfg, "tangent", "tsd")[0] == pytest.approx(np.sqrt(1 - c * c), rel=1e-6)
    assert _const(B, cfg, "tangent", "tim")[0] == pytest.approx(1 / (1 - c), rel=1e-6)
    assert _const(B, cfg, "tangent", "tip")[0] == pytest.approx(1 / (1 + c), rel=1e-6)
    assert np.allclose(_const(B, cfg, "tangent", "tbt")[:2], 0.5 / R, rtol=1e-6)
    assert np.allclose(_const(B, cfg, "tangent", "ax")[:2], R, rtol=1e-6)


def _ball_frame(B, cfg):
    ad = _const(B, cfg, "tangent", "Ad")[: cfg.d]
    q = _const(B, cfg, "tangent", "Q").reshape(3, 3)[: cfg.d, : cfg.d]
    return ad, q


@pytest.mark.parametrize("idx", [3, 4])
def test_rotated_ball_frame(B, idx):
    """Balls: A = Q diag(Ad) Q^T with Q orthonormal (the frame the kernel
    stores points in); ia = 1 / Ad."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx)
    ad, q = _ball_frame(B, cfg)
    assert np.allclose(q.T @ q, np.eye(cfg.d), atol=2e-6)
    assert np.allclose(q @ np.diag(ad) @ q.T, cfg.kt.k_sqrt, atol=2e-6)
    assert np.allclose(_const(B, cfg, "tangent", "ia")[: cfg.d], 1 / ad, rtol=1e-6)


def test_rolling_ball_radius_3d(B):
    """cfg4: rho_b = R min(Ad) / max(Ad)^2 (1 - 1e-6), the smallest curvature
    radius of the whitened ellipsoid |diag(Ad) z| <= R: the rolling ball
    tangent at random boundary points stays inside (sampled)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(4)
    ad, _ = _ball_frame(B, cfg)
    rb = _const(B, cfg, "tangent", "rho_b")[0]
    assert rb == pytest.approx(ad.min() / ad.max() ** 2 * (1 - 1e-6), rel=1e-6)
    rng = np.random.default_rng(3)
    for _ in range(300):
        xb = rng.normal(size=3)
        xb /= np.linalg.norm(xb)
        p = xb / ad
        nrm = -(ad * xb) / np.linalg.norm(ad * xb)
        c = p + rb * nrm
        u = rng.normal(size=(1000, 3))
        u /= np.linalg.norm(u, axis=1)[:, None]
        assert (np.linalg.norm((c + rb * u) * ad, axis=1) <= 1 + 1e-7).all()


def test_annulus_disk_radii(B):
    """cfg3: rho_h = (R - rho) / (2 max Ad) (1 - 1e-6); rho_b = min(R min /
    max^2, that) (1 - 1e-6); mid2 = ((R + rho) / 2)^2; disks of those radii
    tangent to the outer ellipse (inward) and to the hole (outward) at radial
    projections stay inside R and off the hole (sampled)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(3)
    ad, _ = _ball_frame(B, cfg)
    R, rho = 1.0, 0.5
    lim = (R - rho) / (2 * ad.max())
    rb = _const(B, cfg, "tangent", "rho_b")[0]
    rh = _const(B, cfg, "tangent", "rho_h")[0]
    assert rh == pytest.approx(lim * (1 - 1e-6), rel=1e-6)
    assert rb == pytest.approx(min(R * ad.min() / ad.max() ** 2, lim) * (1 - 1e-6), rel=1e-6)
    assert _const(B, cfg, "tangent", "mid2")[0] == pytest.approx(((R + rho) / 2) ** 2, rel=1e-6)
    th = np.linspace(0, 2 * np.pi, 721)
    ring = np.column_stack([np.cos(th), np.sin(th)])
    rng = np.random.default_rng(6)
    for _ in range(300):
        phi = rng.uniform(0, 2 * np.pi)
        xd = np.array([np.cos(phi), np.sin(phi)])
        for rad, sign, r in ((R, -1.0, rb), (rho, 1.0, rh)):
            p = rad * xd / ad
            nrm = sign * (ad * rad * xd) / np.linalg.norm(ad * rad * xd)
            y = p + r * nrm + r * ring
            xr = np.linalg.norm(y * ad, axis=1)
            assert (xr <= R * (1 + 1e-7)).all() and (xr >= rho * (1 - 1e-7)).all()


def test_rolling_disk_blend_and_difference_constants(B):
    """roll2_core's blend constants reproduce the radii exactly and its
    centred-radius margin covers the error bound of the difference forms:
    fl(rho_h + rc_d) == rho_b, nr_d == rho - R, im2 <= 1 / m2, shrink_c >=
    shrink_abs + 5e-7 max|A| R max(1, 1/m2); the plain stop thresholds equal
    the FFMA.SAT ones (bias / scale, exact: the scales are powers of two).
    An anisotropy whose rolling radius is far below the hole-tangent one
    (rho_b << rho_h) keeps the exact blend."""
    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.conductivity import make_tensor

    cfg = configs.get(3)
    for kmat in (None, np.diag([1.0, 400.0]), np.array([[3.0, 1.2], [1.2, 0.9]])):
        if kmat is not None:
            cfg.kt = make_tensor(kmat)
        c = lambda name: np.float32(_const(B, cfg, "tangent", name)[0])
        rb, rh, rcd = c("rho_b"), c("rho_h"), c("rc_d")
        assert np.float32(rh + rcd) == rb and rb <= rh
        assert c("nr_d") == np.float32(np.float32(0.5) - np.float32(1.0))
        m2 = c("m2")
        assert 0 < c("im2") <= np.float32(1.0) / m2
        ad = np.sqrt(np.linalg.eigvalsh(cfg.kt.k_sqrt @ cfg.kt.k_sqrt))
        bound = 5e-7 * max(ad.max(), 1.0) * 1.0 * max(1.0, float(c("im2")))
        assert float(c("shrink_c")) >= float(c("shrink_abs")) + bound * (1 - 1e-3)
        assert c("s2_hi") == np.float32(c("s2_bias") / c("s2_scale"))
        assert c("s2_lo") == np.float32(-c("h2_bias") / c("h2_scale"))
        assert c("s2_hi") == np.float32((1.0 - cfg.eps) ** 2)
        assert c("s2_lo") == np.float32((0.5 + cfg.eps) ** 2)


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_stop_thresholds_are_exact(B, idx):
    """The FFMA.SAT stop tests: stop_scale is a power of two with (e - eps)
    stop_scale >= 1 for the float above eps; for balls s2_bias = fl((R -
    eps)^2) s2_scale with every float below it scaling to >= 1 (so the
    saturated mask is exactly 0/1 at the shell)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx)
    chain = "tangent" if idx > 1 else "max"
    f32 = np.float32
    eps = f32(_const(B, cfg, chain, "eps")[0])
    sc = f32(_const(B, cfg, chain, "stop_scale")[0])
    assert np.log2(sc) == int(np.log2(sc))
    up = np.nextafter(eps, f32(1))
    assert (up - eps) * sc >= 1.0
    if cfg.dom.outer.__class__.__name__ == "Ball":
        s2 = f32(_const(B, cfg, chain, "s2_scale")[0])
        c = f32((1.0 - cfg.eps) ** 2)
        assert f32(_const(B, cfg, chain, "s2_bias")[0]) == c * s2
        below = np.nextafter(c, f32(0))
        assert float(np.float32(np.float32(-below) * s2 + c * s2)) >= 1.0


def test_sheared_box_axes_2d(B):
    """cfg2 on the max chain: u drawn where a_0 = R_0 e1, so A u = (R_0 c,
    R_1 (cos D c + sin D s)) and the stored axes xs_i = x_i / ax_i turn the
    step into xs_0 += r c, xs_1 += r (k c + s): ax = (R_0, R_1 sin D), k =
    cot D (D = angle from a_0 to a_1)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(2)
    R, n = _normals(cfg.kt.k_sqrt)
    dD = np.arctan2(n[1, 1], n[1, 0]) - np.arctan2(n[0, 1], n[0, 0])
    assert _const(B, cfg, "max", "flags")[1] == 1.0  # shear on
    assert np.allclose(_const(B, cfg, "max", "ax")[:2], [R[0], R[1] * np.sin(dD)], rtol=1e-6)
    assert _const(B, cfg, "max", "shk")[0] == pytest.approx(np.cos(dD) / np.sin(dD), rel=1e-5)
