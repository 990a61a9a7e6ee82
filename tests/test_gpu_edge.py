"""Edge cases of the drop-in boundary on the GPU: empty ranges, tiny jobs,
empty families, budget overruns on the FP32 path, replicate offsets across
the 2^32 boundary of the RNG counter, and the size limits.  Conventions
follow the reference driver/kernel (S/backend.py:137-227,
S/_kernel.pyx:376-464; S/ = the reference's src/exitmeasure)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import _native, backend

    _native.require_device(0)
    return backend


@pytest.fixture(scope="module")
def cfg2():
    from paper_2409_03686_b200 import configs

    return configs.get(2)


def _sides(B, cfg):
    return B.pack_side(cfg.fam0, cfg.d, cfg.eps), B.pack_side(cfg.fam1, cfg.d, cfg.eps)


@pytest.mark.parametrize("precision", ["ref64", "fp32"])
def test_zero_replicates(B, cfg2, precision):
    s0, s1 = _sides(B, cfg2)
    r = B.run_accumulate(cfg2.dom, cfg2.kt.k_sqrt, cfg2.poles[:5], cfg2.seed, cfg2.eps, 10**6, 0,
                         s0, s1, precision=precision)
    assert r.raw0.shape == (5, s0.size) and r.raw1.shape == (5, s1.size)
    assert not r.raw0.any() and not r.raw1.any()
    assert not r.steps_sum.any() and not r.steps_max.any()


def test_zero_poles(B, cfg2):
    s0, s1 = _sides(B, cfg2)
    r = B.run_accumulate(cfg2.dom, cfg2.kt.k_sqrt, np.zeros((0, 2)), cfg2.seed, cfg2.eps, 10**6,
                         100, s0, s1, precision="fp32")
    assert r.raw0.shape == (0, s0.size) and r.raw1.shape == (0, s1.size)
    assert r.steps_sum.shape == (0,)


def test_empty_chunk_range(B, cfg2):
    """accumulate_chunk / walk_exits_chunk with rep_start == rep_end leave the
    outputs untouched and report no error (the reference's empty loop)."""
    s0, s1 = _sides(B, cfg2)
    geom = B.pack_geometry(cfg2.dom)
    out0 = np.full(s0.size, 7.0)
    out1 = np.full(s1.size, 3.0)
    res = B.accumulate_chunk(geom.gi, geom.gf, geom.comp_side, cfg2.kt.k_sqrt, cfg2.poles[0], 0,
                             5, 5, cfg2.seed, cfg2.eps, 10**6, s0.anchors, s0.blk, s0.blkf, 0,
                             np.zeros(0), 2, s1.anchors, s1.blk, s1.blkf, 0, np.zeros(0), 2,
                             out0, out1)
    assert tuple(res) == (0, 0, 0, 0, -1)
    assert np.all(out0 == 7.0) and np.all(out1 == 3.0)
    x, steps, comp, err = B.walk_exits_chunk(geom.gi, geom.gf, geom.comp_side, cfg2.kt.k_sqrt,
                                             cfg2.poles[0], 0, 9, 9, cfg2.seed, cfg2.eps, 10**6)
    assert x.shape == (0, 2) and steps.shape == (0,) and comp.shape == (0,) and err == -1


@pytest.mark.parametrize("n_rep", [1, 5, 31, 33])
def test_fp32_tiny_jobs_count_every_walk(B, cfg2, n_rep):
    """Fewer walks than one warp / one block: every walk is counted once."""
    s0, s1 = _sides(B, cfg2)
    r = B.run_accumulate(cfg2.dom, cfg2.kt.k_sqrt, cfg2.poles[:3], cfg2.seed, cfg2.eps, 10**6,
                         n_rep, s0, s1, precision="fp32")
    assert np.all(r.counts.sum(axis=1) == n_rep)
    assert np.all(r.steps_max >= 1) and np.all(r.steps_sum >= n_rep)


def test_empty_family_on_a_used_side_is_rejected(B, cfg2):
    """An exit side with no anchors is a configuration error at the boundary
    (the reference's kernel would write out of bounds)."""
    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.errors import NativeError

    cfg3 = configs.get(3)  # annulus: outer circle -> Gamma0, hole -> Gamma1
    s0 = B.pack_side(None, 2, cfg3.eps)
    _, s1 = _sides(B, cfg3)
    for precision in ("ref64", "fp32"):
        with pytest.raises(NativeError, match="side0"):
            B.run_accumulate(cfg3.dom, cfg3.kt.k_sqrt, cfg3.poles[:2], cfg3.seed, cfg3.eps, 10**6,
                             10, s0, s1, precision=precision)


def test_fp32_budget_error_is_the_smallest_failing_walk(B, cfg2):
    """With a tiny step budget the FP32 run reports the lexicographically
    smallest (pole, replicate) whose walk needs more steps, exactly as the
    reference's job-order scan (S/backend.py:189-192); the step counts come
    from the same walks run through the exits kernel with a large budget."""
    from paper_2409_03686_b200.errors import WalkBudgetError

    s0, s1 = _sides(B, cfg2)
    budget = 6
    poles = cfg2.poles[:4]
    expect = None
    for p in range(len(poles)):
        _, steps, _ = B.run_exits(cfg2.dom, cfg2.kt.k_sqrt, poles[p], p, cfg2.seed, cfg2.eps,
                                  10**6, 64, precision="fp32")
        over = np.nonzero(steps > budget)[0]
        if over.size:
            expect = (p, int(over[0]))
            break
    assert expect is not None
    with pytest.raises(WalkBudgetError) as ei:
        B.run_accumulate(cfg2.dom, cfg2.kt.k_sqrt, poles, cfg2.seed, cfg2.eps, budget, 64, s0, s1,
                         precision="fp32")
    assert (ei.value.pole, ei.value.replicate, ei.value.max_steps) == (*expect, budget)


@pytest.mark.parametrize("rep_start", [0, 1000, 2**32 - 3])
def test_fp32_replicate_ranges_compose(B, cfg2, rep_start):
    """Replicates [a, c) = [a, b) + [b, c) row for row (every walk keyed by
    its own replicate index), including a range across the 2^32 boundary of
    the RNG counter's low word."""
    s0, s1 = _sides(B, cfg2)
    geom = B.pack_geometry(cfg2.dom)
    with B.Plan(geom, cfg2.kt.k_sqrt, cfg2.poles[:4], cfg2.eps, 10**6, s0, s1, "fp32") as plan:
        full = plan.run(cfg2.seed, 40, rep_start).counts.copy()
        a = plan.run(cfg2.seed, 7, rep_start).counts.copy()
        b = plan.run(cfg2.seed, 33, rep_start + 7).counts.copy()
    assert np.array_equal(full, a + b)
    assert np.all(full.sum(axis=1) == 40)


def test_fp32_replicate_limit(B, cfg2):
    """More than 2^31 - 1 replicates per pole in one FP32 run is refused
    before anything is launched (int32 replicate offsets in the kernel)."""
    from paper_2409_03686_b200.errors import NativeError

    s0, s1 = _sides(B, cfg2)
    geom = B.pack_geometry(cfg2.dom)
    with B.Plan(geom, cfg2.kt.k_sqrt, cfg2.poles[:1], cfg2.eps, 10**6, s0, s1, "fp32") as plan:
        with pytest.raises(NativeError, match="2\\^31"):
            plan.run(cfg2.seed, 2**31)


@pytest.mark.parametrize("precision", ["fp32", "ref64"])
def test_plan_cache_reuse_is_exact(B, cfg2, precision):
    """run_accumulate reuses a cached plan for identical inputs: repeated
    calls give identical rows, a new seed or walk count reruns the same plan,
    and changed inputs (poles edited in place) build a new plan."""
    from concurrent.futures import ThreadPoolExecutor

    s0, s1 = _sides(B, cfg2)
    poles = cfg2.poles[:8].copy()
    B.clear_plan_cache()

    def call(seed, n=2000, p=poles):
        return B.run_accumulate(cfg2.dom, cfg2.kt.k_sqrt, p, seed, cfg2.eps, 10**6, n, s0, s1,
                                precision=precision)

    a = call(5)
    assert len(B._PLAN_CACHE) == 1
    b = call(5)
    assert np.array_equal(a.counts, b.counts) and np.array_equal(a.steps_sum, b.steps_sum)
    c = call(6, 3000)
    assert len(B._PLAN_CACHE) == 1 and c.counts.sum() == 8 * 3000
    with B.Plan(B.pack_geometry(cfg2.dom), cfg2.kt.k_sqrt, poles, cfg2.eps, 10**6, s0, s1,
                precision=precision) as plan:
        fresh = plan.run(6, 3000)
    assert np.array_equal(c.counts, fresh.counts)
    # concurrent callers: one takes the cached plan, the others one-shot plans
    with ThreadPoolExecutor(4) as ex:
        outs = list(ex.map(lambda _: call(5), range(4)))
    for o in outs:
        assert np.array_equal(o.counts, a.counts)
    p2 = poles.copy()
    p2[0] *= 0.5
    d = call(5, p=p2)
    assert len(B._PLAN_CACHE) == 2
    assert not np.array_equal(d.counts[0], a.counts[0])
    assert np.array_equal(d.counts[1:], a.counts[1:])
    e = B.run_accumulate(cfg2.dom, cfg2.kt.k_sqrt, poles, 5, cfg2.eps, 10**6, 2000, s0, s1,
                         precision=precision, cache=False)
    assert np.array_equal(e.counts, a.counts) and len(B._PLAN_CACHE) == 2
    B.clear_plan_cache()
    assert len(B._PLAN_CACHE) == 0


@pytest.mark.parametrize("d", [2, 3])
def test_fp32_rolling_chain_pole_at_the_centre(B, d):
    """A pole at the exact centre of a ball (x = 0: |x| and |Ax| vanish in the
    rolling-ball construction) still walks and bins every walk into a valid
    column: exact row sums, and by the symmetry x -> -x of the ellipse /
    ellipsoid the two halves of the boundary get equal mass.  3D: cfg4; 2D:
    cfg1's disk with cfg2's anisotropic K."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(4 if d == 3 else 1)
    k = cfg.kt.k_sqrt if d == 3 else configs.get(2).kt.k_sqrt
    geom = B.pack_geometry(cfg.dom)
    s0, s1 = B.pack_side(cfg.fam0, d, cfg.eps), B.pack_side(cfg.fam1, d, cfg.eps)
    n = 200_000
    with B.Plan(geom, k, np.zeros((1, d)), cfg.eps, 10**6, s0, s1, precision="fp32",
                chain="tangent") as plan:
        assert plan.chain == "tangent"
        r = plan.run(5, n)
    assert int(r.counts.sum()) == n
    half = r.counts.shape[1] // 2
    lower = r.counts[0, half:].sum() / n
    assert abs(lower - 0.5) < 0.01, lower


def test_family_check_under_device_asserts():
    """tools/family_check.py (every walk-kernel family: exact rows, finite
    exits, in-range bins) on the EM_DEBUG build, whose device bounds asserts
    trap on any out-of-range count-row write or work hand-out."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    if not (root / "paper_2409_03686_b200" / "lib" / "libexitmeasure_b200_debug.so").exists():
        pytest.skip("debug library not built")
    env = dict(os.environ, EXITMEASURE_B200_DEBUG="1", EXITMEASURE_B200_AUTOBUILD="0")
    code = ("import runpy, sys; sys.path.insert(0, %r); "
            "from paper_2409_03686_b200 import _native; "
            "assert _native.build_info()['debug'] == '1'; "
            "runpy.run_path(%r, run_name='__main__')") % (str(root), str(root / "tools" / "family_check.py"))
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert "family_check ok" in res.stdout


def test_fp32_rejects_shells_below_its_resolution(B):
    """eps below 2^-20 x the domain scale cannot be reached by FP32 steps that
    keep their rounding margins: the plan refuses it (EM_ERR_UNSUPPORTED)
    instead of stalling every walk at the budget; REF64 runs it."""
    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.errors import NativeError

    cfg = configs.get(1).subset(2, 100)
    s0 = B.pack_side(cfg.fam0, 2, 1e-10)
    s1 = B.pack_side(cfg.fam1, 2, 1e-10)
    with pytest.raises(NativeError, match="ref64"):
        B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, 1, 1e-10, 10**6, 100, s0, s1,
                         precision="fp32")
    r = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, 1, 1e-10, 10**6, 100, s0, s1,
                         precision="ref64")
    assert np.array_equal(r.counts.sum(1), np.full(2, 100))


def test_idw_family_refused_on_integer_rows(B):
    """An IDW weight family has fractional rows: the integer-count entry
    points refuse it (EM_ERR_UNSUPPORTED / ValidationError) instead of
    silently binning to the nearest anchor; run_raw serves it."""
    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.errors import NativeError, ValidationError

    cfg = configs.get(3).subset(2, 64)
    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 2, cfg.eps, "idw", np.full(cfg.fam1.points.shape[0], 0.3), 2)
    import torch

    with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1,
                precision="ref64") as plan:
        counts = torch.zeros((2, plan.n0 + plan.n1), dtype=torch.int64, device="cuda")
        stats = torch.zeros((3, 2), dtype=torch.int64, device="cuda")
        with pytest.raises(ValidationError):
            plan.run_device(1, 64, counts.data_ptr(), stats.data_ptr())
        r = plan.run(1, 64)  # routes to run_raw
        assert np.allclose(r.raw0.sum(1) + r.raw1.sum(1), 64)
    # the C ABI's integer entry point refuses it outright
    from paper_2409_03686_b200 import _native as N

    m = B._Marshal()
    g = m.geometry(geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt)
    ms0, ms1 = m.sidepack(s0), m.sidepack(s1)
    out = N.EmOutputs(*[m.arr(np.zeros(n, np.int64), np.int64).ctypes.data
                        for n in (2 * (s0.size + s1.size), 2, 2, 2)], -1, -1)
    import ctypes

    opt = N.EmOptions(N.EM_PREC_REF64, N.EM_CHAIN_WOE, 0, 0, 0, 0)
    pl = m.arr(cfg.poles, np.float64)
    rc = N.lib().em_run_accumulate(ctypes.byref(g), ctypes.byref(ms0), ctypes.byref(ms1),
                                   N.ptr(pl), None, 2, 1, cfg.eps, 10**6, 64,
                                   ctypes.byref(opt), ctypes.byref(out))
    assert rc == N.EM_ERR_UNSUPPORTED, rc
    with pytest.raises(NativeError):
        N.check(rc, "em_run_accumulate")


@pytest.mark.parametrize("precision", ["fp32", "ref64"])
def test_float64_rows_from_the_device(B, precision):
    """em_plan_run_host_f64: the reference's float64 raw rows converted on
    the device equal the int64 counts exactly (the plugin's path)."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(3).subset(8, 3000)
    s0 = B.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = B.pack_side(cfg.fam1, 2, cfg.eps)
    a = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, 5, cfg.eps, 10**6, cfg.n_rep, s0, s1,
                         precision=precision, cache=False)
    f = B.run_accumulate(cfg.dom, cfg.kt.k_sqrt, cfg.poles, 5, cfg.eps, 10**6, cfg.n_rep, s0, s1,
                         precision=precision, cache=False, rows="float64")
    assert f.counts is None and f.raw0.dtype == np.float64
    assert np.array_equal(f.raw0, a.counts[:, : s0.size].astype(np.float64))
    assert np.array_equal(f.raw1, a.counts[:, s0.size:].astype(np.float64))
    assert np.array_equal(f.steps_sum, a.steps_sum) and np.array_equal(f.steps_max, a.steps_max)
