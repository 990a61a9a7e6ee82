"""The packed two-walks-per-lane kernel equals the one-walk-per-lane kernel.

FP32 counts on the 2D ball's rolling-disk chain (cfg3, the headline) run two
walks per lane with Blackwell's packed FP32 instructions (FFMA2 / FMUL2 /
FADD2, csrc/walk_f32x2.cu).  Both kernels instantiate ONE operation tree
(csrc/walk_f32_dev.cuh roll2_core, explicit round-to-nearest operations), key
every walk's random stream by (seed, global pole id, replicate) and
accumulate integers, so counts and step statistics must agree EXACTLY --
on every scheduler, on row shards, with replicate offsets, and in the budget
error they report.  The one-walk kernel's sampler is the one the closed-form
tests pin (tests/test_gpu_closed_form.py); this file carries that evidence
over to the packed kernel bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import _native, backend

    _native.require_device(0)
    return backend


def _plans(B, cfg, pole_ids=None, max_steps=10**6, sched=0):
    from paper_2409_03686_b200 import _native

    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    mk = lambda fl: B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, max_steps, s0, s1,
                           precision="fp32", pole_ids=pole_ids, flags=fl | sched)
    # the packed kernel at every size (by default runs below 2e6 walks take
    # the one-walk kernel) against the one-walk kernel
    return mk(_native.EM_FLAG_TWO_WALKS_PER_LANE), mk(_native.EM_FLAG_ONE_WALK_PER_LANE)


def _same(a, b):
    assert np.array_equal(a.counts, b.counts)
    assert np.array_equal(a.steps_sum, b.steps_sum)
    assert np.array_equal(a.steps_sq_sum, b.steps_sq_sum)
    assert np.array_equal(a.steps_max, b.steps_max)


@pytest.mark.parametrize("n_poles,n_rep", [(1024, 20_000), (64, 300_000), (7, 1), (3, 65), (1, 5_000)])
def test_packed_equals_one_walk_per_lane_cfg3(B, n_poles, n_rep):
    from paper_2409_03686_b200 import configs

    cfg = configs.get(3).subset(n_poles)
    p2, p1 = _plans(B, cfg)
    with p2, p1:
        assert p2.walks_per_lane() == 2 and p1.walks_per_lane() == 1
        r2, r1 = p2.run(cfg.seed, n_rep), p1.run(cfg.seed, n_rep)
        assert p2.last_walks_per_lane() == 2 and p1.last_walks_per_lane() == 1
    assert np.array_equal(r2.counts.sum(1), np.full(cfg.n_poles, n_rep))
    _same(r2, r1)


def test_default_kernel_follows_job_size(B):
    """Default flags: runs of >= 2e6 walks take the packed kernel, smaller
    ones the one-walk kernel (identical counts either way)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(3).subset(64)
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1, precision="fp32") as plan:
        assert plan.walks_per_lane() == 2
        plan.run(cfg.seed, 1000)
        assert plan.last_walks_per_lane() == 1
        plan.run(cfg.seed, 40_000)
        assert plan.last_walks_per_lane() == 2
    cfg5 = configs.get(5).subset(8)
    with B.Plan(B.pack_geometry(cfg5.dom), cfg5.kt.k_sqrt, cfg5.poles, cfg5.eps, 10**6,
                B.pack_side(cfg5.fam0, 3, cfg5.eps), B.pack_side(cfg5.fam1, 3, cfg5.eps),
                precision="fp32") as plan:
        assert plan.walks_per_lane() == 1  # no packed kernel for the L-box's table-driven chain


@pytest.mark.parametrize("n_poles,n_rep", [(256, 100_000), (256, 3_000), (5, 77)])
def test_packed_equals_one_walk_per_lane_cfg2(B, n_poles, n_rep):
    """The 2D box on tangent balls (tang2_core), square-arc binner."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(2).subset(n_poles)
    p2, p1 = _plans(B, cfg)
    with p2, p1:
        assert p2.walks_per_lane() == 2 and p1.walks_per_lane() == 1
        r2, r1 = p2.run(cfg.seed, n_rep), p1.run(cfg.seed, n_rep)
    assert np.array_equal(r2.counts.sum(1), np.full(cfg.n_poles, n_rep))
    _same(r2, r1)


@pytest.mark.parametrize("n_poles,n_rep", [(1024, 5_000), (32, 100_000), (3, 33)])
def test_packed_equals_one_walk_per_lane_cfg4(B, n_poles, n_rep):
    """The 3D ball on rolling balls (roll3_core), candidate-grid binner."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(4).subset(n_poles)
    p2, p1 = _plans(B, cfg)
    with p2, p1:
        assert p2.walks_per_lane() == 2 and p1.walks_per_lane() == 1
        r2, r1 = p2.run(cfg.seed, n_rep), p1.run(cfg.seed, n_rep)
        assert p2.last_walks_per_lane() == 2 and p1.last_walks_per_lane() == 1
    assert np.array_equal(r2.counts.sum(1), np.full(cfg.n_poles, n_rep))
    _same(r2, r1)


def test_packed_box_off_origin_grid_binner_and_budget(B):
    """An off-origin rectangle with a strongly anisotropic K and an
    unstructured anchor family (candidate-grid binner); then a step budget
    the walks overrun."""
    from paper_2409_03686_b200 import _native
    from paper_2409_03686_b200.conductivity import make_tensor
    from paper_2409_03686_b200.errors import WalkBudgetError
    from paper_2409_03686_b200.geometry import Box, Domain, generic_points, square_points

    dom = Domain(2, Box(np.array([1.5, -0.25]), 0.75), (), frozenset())
    kt = make_tensor([[4.0, 1.5], [1.5, 1.0]])
    pts = square_points(np.array([1.5, -0.25]), 0.75, 200, component=0, phase=0.5).points
    fam1 = generic_points(pts, component=0)
    rng = np.random.default_rng(5)
    poles = np.array([1.5, -0.25]) + rng.uniform(-0.7, 0.7, size=(40, 2))
    geom = B.pack_geometry(dom)
    s0 = B.pack_side(None, 2, 1e-5)
    s1 = B.pack_side(fam1, 2, 1e-5)
    out = []
    for fl in (_native.EM_FLAG_TWO_WALKS_PER_LANE, _native.EM_FLAG_ONE_WALK_PER_LANE):
        with B.Plan(geom, kt.k_sqrt, poles, 1e-5, 10**6, s0, s1, precision="fp32", flags=fl) as plan:
            out.append((plan.run(11, 30_000), plan.walks_per_lane()))
    assert out[0][1] == 2 and out[1][1] == 1
    _same(out[0][0], out[1][0])
    errs = []
    for fl in (_native.EM_FLAG_TWO_WALKS_PER_LANE, _native.EM_FLAG_ONE_WALK_PER_LANE):
        with B.Plan(geom, kt.k_sqrt, poles, 1e-5, 2, s0, s1, precision="fp32", flags=fl) as plan:
            with pytest.raises(WalkBudgetError) as ei:
                plan.run(11, 4096)
            errs.append((ei.value.pole, ei.value.replicate))
    assert errs[0] == errs[1]


def test_packed_equals_one_walk_per_lane_schedulers_shards_offsets(B):
    """Pole blocks (shared-memory histograms) and pole-cycling warps, on a
    row shard with global pole ids and a replicate offset beyond 2^32."""
    from paper_2409_03686_b200 import _native, configs

    cfg = configs.get(3).subset(16)
    ids = np.arange(3, 64, 4)
    ref = None
    for sched in (_native.EM_FLAG_PERSISTENT, _native.EM_FLAG_POLE_BLOCKS):
        p2, p1 = _plans(B, cfg, pole_ids=ids, sched=sched)
        with p2, p1:
            r2 = p2.run(cfg.seed, 40_000, (1 << 32) + 12_345)
            r1 = p1.run(cfg.seed, 40_000, (1 << 32) + 12_345)
            assert p2.walks_per_lane() == 2
            assert p2.last_scheduler() == p1.last_scheduler()
        _same(r2, r1)
        if ref is not None:
            _same(r2, ref)
        ref = r2


def test_packed_budget_error_equals_one_walk_per_lane(B):
    """A step budget the walks overrun (the per-step budget path of the packed
    kernel): the same lexicographically first (global pole, replicate)."""
    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.errors import WalkBudgetError

    cfg = configs.get(3).subset(5)
    ids = np.array([9, 4, 11, 2, 40])
    errs = []
    for plan in _plans(B, cfg, pole_ids=ids, max_steps=3):
        with plan:
            with pytest.raises(WalkBudgetError) as ei:
                plan.run(cfg.seed, 8192)
            errs.append((ei.value.pole, ei.value.replicate))
    assert errs[0] == errs[1] and errs[0][0] == 9
    # a budget only the long walks overrun: some batches take the per-step
    # path, the rest the fast path; results must still agree where no walk fails
    p2, p1 = _plans(B, cfg, max_steps=64)
    with p2, p1:
        try:
            r2 = p2.run(cfg.seed, 2000)
        except WalkBudgetError as e:
            r2 = (e.pole, e.replicate)
        try:
            r1 = p1.run(cfg.seed, 2000)
        except WalkBudgetError as e:
            r1 = (e.pole, e.replicate)
    if isinstance(r2, tuple) or isinstance(r1, tuple):
        assert r2 == r1
    else:
        _same(r2, r1)


def test_packed_disc_without_hole_equals_one_walk_per_lane(B):
    """The no-hole instantiation (2D ball, K != I, rolling disks): cfg3's K on
    the unit disc with 256 arcs."""
    from paper_2409_03686_b200 import _native, configs
    from paper_2409_03686_b200.geometry import Ball, Domain, circle_points

    cfg = configs.get(3)
    dom = Domain(2, Ball(np.zeros(2), 1.0), (), frozenset())
    fam1 = circle_points(np.zeros(2), 1.0, 256, component=0, phase=0.5)
    geom = B.pack_geometry(dom)
    s0 = B.pack_side(None, 2, cfg.eps)
    s1 = B.pack_side(fam1, 2, cfg.eps)
    poles = 0.8 * cfg.poles[:48]
    out = []
    for fl in (_native.EM_FLAG_TWO_WALKS_PER_LANE, _native.EM_FLAG_ONE_WALK_PER_LANE):
        with B.Plan(geom, cfg.kt.k_sqrt, poles, cfg.eps, 10**6, s0, s1, precision="fp32",
                    flags=fl) as plan:
            out.append((plan.run(cfg.seed, 50_000), plan.walks_per_lane()))
    assert out[0][1] == 2 and out[1][1] == 1
    assert np.array_equal(out[0][0].counts.sum(1), np.full(48, 50_000))
    _same(out[0][0], out[1][0])


def _strong_anisotropy_case(name):
    """Rolling-chain geometries with strongly anisotropic K (the difference-form
    centred radius with 1 / m2 up to 5 and |A| up to 5.5, rolling radii far
    below the hole-tangent one, eigenvalues below 1)."""
    from paper_2409_03686_b200.conductivity import make_tensor
    from paper_2409_03686_b200.geometry import (Ball, Domain, circle_points, fibonacci_sphere,
                                                generic_points)

    if name == "annulus30":
        c, s = np.cos(0.4), np.sin(0.4)
        rot = np.array([[c, -s], [s, c]])
        dom = Domain(2, Ball(np.zeros(2), 1.0), (Ball(np.zeros(2), 0.4),), frozenset({0}))
        kt = make_tensor(rot @ np.diag([1.0, 30.0]) @ rot.T)
        f0 = circle_points(np.zeros(2), 1.0, 96, component=0)
        f1 = circle_points(np.zeros(2), 0.4, 48, component=1)
        poles = np.array([[0.7, 0.1], [-0.2, 0.55], [0.05, -0.9], [-0.45, -0.1]])
        return dom, kt, f0, f1, poles
    if name == "disc_small_eig":
        dom = Domain(2, Ball(np.array([0.3, -0.2]), 0.8), (), frozenset())
        kt = make_tensor(np.array([[0.2, 0.0], [0.0, 6.0]]))
        f1 = circle_points(np.array([0.3, -0.2]), 0.8, 64, component=0, phase=0.5)
        poles = np.array([[0.3, -0.2], [0.8, 0.1], [0.2, 0.45]])
        return dom, kt, None, f1, poles
    dom = Domain(3, Ball(np.zeros(3), 1.0), (), frozenset())
    kt = make_tensor(np.diag([0.3, 1.0, 9.0]))
    f1 = generic_points(fibonacci_sphere(120, 1.0), component=0)
    poles = np.array([[0.0, 0.0, 0.0], [0.6, -0.3, 0.2], [-0.1, 0.2, -0.85]])
    return dom, kt, None, f1, poles


@pytest.mark.parametrize("name", ["annulus30", "disc_small_eig", "ball9"])
def test_packed_rolling_chains_strong_anisotropy_vs_oracle(B, oracle, name):
    """The packed kernel on strongly anisotropic rolling-chain geometries:
    equal to the one-walk kernel bit for bit, and statistically equal to the
    oracle's FP64 reference chain (entry-wise exact binomial tests at
    family-wise level 1e-4, row chi^2 homogeneity)."""
    from helpers import P_Z4, exact_two_sample_p, exceed_quantile, row_chi2_pvalues
    from paper_2409_03686_b200 import _native

    dom, kt, f0, f1, poles = _strong_anisotropy_case(name)
    d = poles.shape[1]
    eps = 1e-5
    geom = B.pack_geometry(dom)
    s0, s1 = B.pack_side(f0, d, eps), B.pack_side(f1, d, eps)
    n_gpu, n_ref = 400_000, 20_000
    res = []
    for fl in (_native.EM_FLAG_TWO_WALKS_PER_LANE, _native.EM_FLAG_ONE_WALK_PER_LANE):
        with B.Plan(geom, kt.k_sqrt, poles, eps, 10**6, s0, s1, precision="fp32", flags=fl) as plan:
            assert plan.chain == "tangent"
            res.append((plan.run(77, n_gpu), plan.last_walks_per_lane()))
    assert res[0][1] == 2 and res[1][1] == 1
    _same(res[0][0], res[1][0])
    r = res[0][0]
    assert np.array_equal(r.counts.sum(1), np.full(len(poles), n_gpu))

    def generic(sd):  # brute-force Voronoi blocks: the oracle's exact binning
        return (sd.anchors, np.array([[0, 0, sd.size]]), np.zeros((1, 4)))

    raw0, raw1, *_ = oracle.run_accumulate_packed(geom.gi, geom.gf, geom.comp_side, kt.k_sqrt, poles,
                                                  5, eps, 10**6, n_ref, generic(s0), generic(s1))
    ref = np.concatenate([raw0, raw1], axis=1)
    p = exact_two_sample_p(r.counts, n_gpu, ref, n_ref)
    m = p.size
    worst = np.unravel_index(p.argmin(), p.shape)
    assert p.min() >= 1e-4 / m, (p.min(), worst, r.counts[worst], ref[worst])
    assert int((p < P_Z4).sum()) <= exceed_quantile(m, q=0.99999)
    rows = row_chi2_pvalues(r.counts, n_gpu, ref, n_ref)
    assert rows.min() > 1e-5 / len(rows), rows.min()
    # the tangent chain engaged: far fewer steps than the reference chain's
    assert r.steps_sum.sum() / (len(poles) * n_gpu) < 14
