"""The two FP32 schedulers give identical results.

North_star's per-block shared-memory histograms (one block per (pole,
replicate range), warp-aggregated __match_any_sync adds, one int64 flush per
block; the default where the rows exceed half the L2, e.g. cfg5) against the
pole-cycling persistent warps with one int64 atomic per exit (the default
for L2-resident rows).  Every walk's random stream is keyed by (seed, pole,
replicate) and all accumulation is integer, so counts and step statistics
must agree EXACTLY (the reference's own chunking-invariance contract,
T/test_backend.py:118-137)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_2409_03686_b200 import _native, backend

    _native.require_device(0)
    return backend


def _all(B, cfg, n_rep, pole_ids=None, rep_start=0, max_steps=10**6):
    from paper_2409_03686_b200 import _native

    geom = B.pack_geometry(cfg.dom)
    s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
    s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
    out = {}
    for name, flags in (("blocks", _native.EM_FLAG_POLE_BLOCKS),
                        ("persistent", _native.EM_FLAG_PERSISTENT)):
        with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, max_steps, s0, s1,
                    precision="fp32", pole_ids=pole_ids, flags=flags) as plan:
            try:
                r = plan.run(cfg.seed, n_rep, rep_start)
                out[name] = (r, plan.last_scheduler())
            except Exception as e:  # budget errors are compared too
                out[name] = (e, plan.last_scheduler())
    return out


@pytest.mark.parametrize("idx,n_poles,n_rep", [(3, 12, 50_000), (4, 6, 40_000), (5, 4, 20_000)])
def test_pole_block_scheduler_equals_persistent(B, idx, n_poles, n_rep):
    from paper_2409_03686_b200 import configs

    cfg = configs.get(idx).subset(n_poles)
    out = _all(B, cfg, n_rep)
    (rp, sp) = out["persistent"]
    assert sp.startswith("persistent"), sp
    assert np.array_equal(rp.counts.sum(1), np.full(cfg.n_poles, n_rep))
    for name, want in (("blocks", "pole-blocks"),):
        rb, sb = out[name]
        assert sb == want, (name, sb)
        assert np.array_equal(rb.counts, rp.counts), name
        assert np.array_equal(rb.steps_sum, rp.steps_sum), name
        assert np.array_equal(rb.steps_sq_sum, rp.steps_sq_sum), name
        assert np.array_equal(rb.steps_max, rp.steps_max), name


def test_pole_block_scheduler_shards_and_offsets(B):
    """Row shards (global pole ids) and replicate offsets key the same
    streams on both schedulers."""
    from paper_2409_03686_b200 import configs

    cfg = configs.get(3).subset(16)
    ids = np.arange(1, 32, 2)
    out = _all(B, cfg, 30_000, pole_ids=ids, rep_start=123_457)
    rp, _ = out["persistent"]
    for name in ("blocks",):
        rb, _ = out[name]
        assert np.array_equal(rb.counts, rp.counts), name
        assert np.array_equal(rb.steps_sum, rp.steps_sum), name


def test_pole_block_scheduler_budget_error(B):
    """A step budget the walks overrun: both schedulers report the same
    lexicographically first (global pole, replicate)."""
    from paper_2409_03686_b200 import configs
    from paper_2409_03686_b200.errors import WalkBudgetError

    cfg = configs.get(4).subset(5)
    ids = np.array([7, 3, 11, 2, 40])
    out = _all(B, cfg, 8192, pole_ids=ids, max_steps=3)
    ep, _ = out["persistent"]
    assert isinstance(ep, WalkBudgetError) and ep.pole == 7  # first row of the plan
    for name in ("blocks",):
        eb, _ = out[name]
        assert isinstance(eb, WalkBudgetError), name
        assert (eb.pole, eb.replicate) == (ep.pole, ep.replicate), name


def test_default_scheduler_follows_row_size(B):
    """Defaults: pole blocks for cfg5's 256 MiB of rows, pole-cycling warps for
    cfg3's 8 MiB (L2-resident)."""
    from paper_2409_03686_b200 import configs

    for idx, want in ((5, "pole-blocks"), (3, "persistent")):
        cfg = configs.get(idx)
        geom = B.pack_geometry(cfg.dom)
        s0 = B.pack_side(cfg.fam0, cfg.d, cfg.eps)
        s1 = B.pack_side(cfg.fam1, cfg.d, cfg.eps)
        with B.Plan(geom, cfg.kt.k_sqrt, cfg.poles, cfg.eps, 10**6, s0, s1,
                    precision="fp32") as plan:
            r = plan.run(cfg.seed, 4096)
            assert plan.last_scheduler() == want, (idx, plan.last_scheduler())
        assert np.array_equal(r.counts.sum(1), np.full(cfg.n_poles, 4096))
