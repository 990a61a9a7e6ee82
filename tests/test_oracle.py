"""The CPU oracle (oracle/em_oracle.c) pinned against the reference's golden
vectors -- no GPU needed.  If the oracle drifts from the reference, every GPU
parity claim built on it is void, so these run on every CPU test pass."""

import numpy as np
import pytest

from helpers import CASE_NAMES, case, side_tuple


def test_philox_matches_numpy_golden(oracle, golden_philox):
    """numpy.random.Philox pre-increments its counter (T/test_rng.py:7-24)."""
    g = golden_philox
    for key, ctr, raw in zip(g["keys"], g["counters"], g["numpy_raw"]):
        c = [int(v) for v in ctr]
        c[0] = (c[0] + 1) % 2**64
        if c[0] == 0:
            c[1] = (c[1] + 1) % 2**64
        assert oracle.philox4x64(int(key), *c) == [int(w) for w in raw]


def test_philox_matches_reference_rng(oracle, golden_philox):
    g = golden_philox
    for row, out in zip(g["ref_in"], g["ref_out"]):
        s, k1, c0, c1, c2, c3 = (int(v) for v in row)
        assert oracle.philox4x64(s, c0, c1, c2, c3, key1=k1) == [int(w) for w in out]


@pytest.mark.parametrize("name", CASE_NAMES)
def test_walk_exits_bit_identical_to_reference(oracle, golden_cases, name):
    c = case(golden_cases, name)
    x, st, comp, err = oracle.walk_exits_chunk(c["gi"], c["gf"], c["comp_side"], c["ksqrt"],
                                               c["pole"], 2, 10, 210, 99, float(c["eps"]),
                                               10**6)
    assert err == -1
    assert np.array_equal(x, c["x"])
    assert np.array_equal(st, c["steps"])
    assert np.array_equal(comp, c["comp"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_accumulate_bit_identical_to_reference(oracle, golden_cases, name):
    c = case(golden_cases, name)
    o0 = np.zeros(c["a0"].shape[0])
    o1 = np.zeros(c["a1"].shape[0])
    stats = oracle.accumulate_chunk(c["gi"], c["gf"], c["comp_side"], c["ksqrt"], c["pole"], 0,
                                    0, 3000, 7, float(c["eps"]), 10**6,
                                    *side_tuple(c, 0), *side_tuple(c, 1), o0, o1)
    assert np.array_equal(o0, c["out0"]) and np.array_equal(o1, c["out1"])
    assert list(stats) == [int(v) for v in c["stats"]]
    assert o0.sum() + o1.sum() == 3000.0


def test_budget_error_first_replicate(oracle, golden_cases):
    c = case(golden_cases, "annulus")
    res = oracle.accumulate_chunk(c["gi"], c["gf"], c["comp_side"], np.eye(2),
                                  np.array([0.95, 0.0]), 0, 0, 50, 1, 1e-10, 2,
                                  *side_tuple(c, 0), *side_tuple(c, 1),
                                  np.zeros(c["a0"].shape[0]), np.zeros(c["a1"].shape[0]))
    assert res[4] == int(golden_cases["budget_err"]) >= 0


def _cfg_inputs(g, idx):
    from paper_2409_03686_b200 import backend, configs

    pre = f"cfg{idx}."
    n_poles = g[pre + "poles"].shape[0]
    cfg = configs.get(idx).subset(n_poles, int(g[pre + "n_rep"]))
    return cfg, backend


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_config_packing_matches_reference_expression(golden_cfg, idx):
    """The package's BASELINE configs hold exactly the poles/anchors/K^{1/2}
    the reference expression was run on."""
    cfg, backend = _cfg_inputs(golden_cfg, idx)
    pre = f"cfg{idx}."
    assert np.array_equal(cfg.poles, golden_cfg[pre + "poles"])
    assert np.allclose(cfg.kt.k_sqrt, golden_cfg[pre + "ksqrt"], rtol=0, atol=1e-15)
    if idx != 3:
        assert np.array_equal(np.ascontiguousarray(cfg.fam1.points), golden_cfg[pre + "anchors1"])


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_oracle_run_accumulate_matches_reference(oracle, golden_cfg, idx):
    """oracle.run_accumulate (S/backend.py:147-199 restated) on the reference
    expression reproduces the reference's count rows bit for bit."""
    cfg, backend = _cfg_inputs(golden_cfg, idx)
    pre = f"cfg{idx}."
    geom = backend.pack_geometry(cfg.dom)
    if idx == 3:
        s0 = backend.pack_side(cfg.fam0, 2, cfg.eps)
        s1 = backend.pack_side(cfg.fam1, 2, cfg.eps)
        side0 = (s0.anchors, s0.blk, s0.blkf)
        side1 = (s1.anchors, s1.blk, s1.blkf)
    else:
        a1 = golden_cfg[pre + "anchors1"]
        side0 = (np.zeros((0, cfg.d)), np.zeros((1, 3), np.int64), np.zeros((1, 4)))
        side1 = (a1, np.array([[0, 0, a1.shape[0]]]), np.zeros((1, 4)))
    raw0, raw1, ss, sq, sm, fb, err = oracle.run_accumulate_packed(
        geom.gi, geom.gf, geom.comp_side, golden_cfg[pre + "ksqrt"], golden_cfg[pre + "poles"],
        int(golden_cfg[pre + "seed"]), float(golden_cfg[pre + "eps"]), 10**6,
        int(golden_cfg[pre + "n_rep"]), side0, side1)
    assert err is None
    assert np.array_equal(raw0, golden_cfg[pre + "raw0"])
    assert np.array_equal(raw1, golden_cfg[pre + "raw1"])
    assert np.array_equal(ss, golden_cfg[pre + "steps_sum"])
    assert np.array_equal(sq, golden_cfg[pre + "steps_sq"])
    assert np.array_equal(sm, golden_cfg[pre + "steps_max"])


def test_oracle_thread_count_invariance(oracle, golden_cfg):
    cfg, backend = _cfg_inputs(golden_cfg, 3)
    geom = backend.pack_geometry(cfg.dom)
    s0 = backend.pack_side(cfg.fam0, 2, cfg.eps)
    s1 = backend.pack_side(cfg.fam1, 2, cfg.eps)
    args = (geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt, cfg.poles[:8], 5, cfg.eps, 10**6,
            9000, (s0.anchors, s0.blk, s0.blkf), (s1.anchors, s1.blk, s1.blkf))
    a = oracle.run_accumulate_packed(*args, threads=1)
    b = oracle.run_accumulate_packed(*args, threads=3)
    for x, y in zip(a[:5], b[:5]):
        assert np.array_equal(x, y)


def test_lbox_distance_and_walks(oracle):
    """cfg5 extension (parity unpinned by the reference: structural checks).
    Exact L-box distance at known points; walks stay in the closure; every
    walk lands in one cell; the notch faces are component 1 / Gamma1."""
    from paper_2409_03686_b200 import backend, configs
    from paper_2409_03686_b200.geometry import dist_to_boundary

    cfg = configs.get(5).subset(6, 300)
    geom = backend.pack_geometry(cfg.dom)
    for p, expect in [((0.25, 0.25, 0.5), 0.25), ((0.45, 0.8, 0.5), 0.05),
                      ((0.4, 0.4, 0.5), 0.02 ** 0.5), ((0.49, 0.49, 0.98), 0.0002 ** 0.5),
                      ((0.75, 0.25, 0.02), 0.02)]:
        got = oracle.signed_dist(geom.gi, geom.gf, np.array(p))
        assert got == pytest.approx(expect, abs=1e-14)
        assert dist_to_boundary(cfg.dom, np.array(p)) == pytest.approx(expect, abs=1e-14)
    assert oracle.owner_component(geom.gi, geom.gf, np.array([0.45, 0.8, 0.5])) == 1
    assert oracle.owner_component(geom.gi, geom.gf, np.array([0.02, 0.3, 0.5])) == 0
    x, st, comp, err = oracle.walk_exits_chunk(geom.gi, geom.gf, geom.comp_side,
                                               cfg.kt.k_sqrt, cfg.poles[0], 0, 0, 400,
                                               cfg.seed, cfg.eps, 10**6)
    assert err == -1
    sd = np.array([oracle.signed_dist(geom.gi, geom.gf, p) for p in x])
    assert sd.min() >= -1e-12 and sd.max() <= cfg.eps
    s0 = backend.pack_side(cfg.fam0, 3, cfg.eps)
    s1 = backend.pack_side(cfg.fam1, 3, cfg.eps)
    raw0, raw1, ss, *_ = oracle.run_accumulate_packed(
        geom.gi, geom.gf, geom.comp_side, cfg.kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6,
        cfg.n_rep, (s0.anchors, s0.blk, s0.blkf), (s1.anchors, s1.blk, s1.blkf))
    assert np.array_equal(raw0.sum(1) + raw1.sum(1), np.full(6, 300.0))


def _idw_sides(c):
    return ((c["a0"], c["blk0"], c["blkf0"], 1, c["r0"], 3),
            (c["a1"], c["blk1"], c["blkf1"], 1, c["r1"], 2))


@pytest.mark.parametrize("name", ["annulus", "square_hole"])
def test_idw_bit_identical_to_reference(oracle, golden_idw, name):
    """IDW families (S/_kernel.pyx:323-369): the chunk contract accumulating
    in place from non-zero rows, and the driver's per-8192-chunk partials
    merged in job order -- both bit for bit."""
    c = case(golden_idw, "idw_" + name)
    s0, s1 = _idw_sides(c)
    o0, o1 = c["init0"].copy(), c["init1"].copy()
    st = oracle.accumulate_chunk(c["gi"], c["gf"], c["comp_side"], c["ksqrt"], c["pole"], 0, 0,
                                 3000, 7, float(c["eps"]), 10**6, *s0, *s1, o0, o1)
    assert np.array_equal(o0, c["out0"]) and np.array_equal(o1, c["out1"])
    assert list(st) == [int(v) for v in c["stats"]]
    raw0, raw1, ss, _, _, fb, err = oracle.run_accumulate_packed(
        c["gi"], c["gf"], c["comp_side"], c["ksqrt"], c["poles2"], 11, float(c["eps"]), 10**6,
        10000, s0, s1, threads=3)
    assert err is None
    assert np.array_equal(raw0, c["raw0"]) and np.array_equal(raw1, c["raw1"])
    assert np.array_equal(ss, c["rsteps"]) and fb == int(c["rfb"])
