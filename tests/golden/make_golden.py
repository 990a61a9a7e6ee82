"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs in the build container only (it imports the reference package, which
does not exist on the GPU box): the compiled reference from oracle/_ref
(oracle/build_ref.sh) if present, else /root/reference/pkg/src with its
bit-identical numpy fallback.  The fixtures it writes are small .npz files
that travel with the repo; tests compare the C oracle (CPU, `-m "not gpu"`)
and the CUDA library (`-m gpu`) against them.

Fixtures:
  philox.npz      numpy.random.Philox raw blocks (the reference's own golden,
                  T/test_rng.py:7-24) + reference philox4x64 on extra counters
  cases.npz       the six geometry/K cases of T/test_backend.py:65-72:
                  walk_exits_chunk and accumulate_chunk outputs of the
                  reference kernel, plus a budget-error case
  idw.npz         IDW families (annulus, square_hole): accumulate_chunk from
                  non-zero initial rows, and run_accumulate over 2 x 10000
                  walks (per-8192-chunk partial sums)
  baseline_cfg.npz  BASELINE cfg1-cfg4 in the reference expression
                   at reduced size: run_accumulate
                  count rows and step statistics

Usage: python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent


def _import_reference():
    ref = ROOT / "oracle" / "_ref"
    if (ref / "exitmeasure").exists():
        sys.path.insert(0, str(ref))
    else:
        os.environ.setdefault("EXITMEASURE_BACKEND", "fallback")
        sys.path.insert(0, "/root/reference/pkg/src")
    import exitmeasure  # noqa: F401
    from exitmeasure import backend

    return backend


def _sides(backend, dom, eps):
    from exitmeasure.geometry import side_points

    d = dom.dimension
    anchors1 = side_points(dom, "gamma1", [60] * len(dom.gamma1))
    side1 = backend.pack_side(anchors1, d, eps)
    if dom.gamma0:
        side0 = backend.pack_side(side_points(dom, "gamma0", [80 * len(dom.gamma0)]), d, eps)
    else:
        side0 = backend.pack_side(None, d, eps)
    return side0, side1


def main():
    backend = _import_reference()
    from exitmeasure.conductivity import identity_tensor, make_tensor
    from exitmeasure.geometry import Ball, Box, BoundaryPointSet, catalog, make_domain
    from exitmeasure.problems import ANISO_K
    from exitmeasure.rng import philox4x64

    impl = backend._impl
    print("reference backend:", backend.BACKEND)

    # ---- philox ----
    keys, ctrs, raws = [], [], []
    for key, ctr in [(123456789, (0, 0, 0, 0)), (7, (5, 0, 42, 99)),
                     (2**63 + 11, (2**64 - 1, 3, 1, 2**50)), (20240905, (17, 0, 9999, 31))]:
        bg = np.random.Philox(counter=np.array(ctr, dtype=np.uint64),
                              key=np.array([key, 0], dtype=np.uint64))
        raws.append(bg.random_raw(4))
        keys.append(key)
        ctrs.append(ctr)
    extra_in = np.array([[s, 0, dr, 0, rep, pole] for s, dr, rep, pole in
                         [(99, 0, 10, 2), (99, 5, 2009, 2), (7, 3, 2999, 0), (1, 0, 0, 0),
                          (2**64 - 1, 2**40, 7, 2**33)]], dtype=np.uint64)
    extra_out = np.array([[int(w) for w in philox4x64(*[np.uint64(v) for v in row])]
                          for row in extra_in], dtype=np.uint64)
    np.savez_compressed(OUT / "philox.npz", keys=np.array(keys, dtype=np.uint64),
                        counters=np.array(ctrs, dtype=np.uint64),
                        numpy_raw=np.array(raws, dtype=np.uint64),
                        ref_in=extra_in, ref_out=extra_out)

    # ---- reference test cases (T/test_backend.py:65-72) ----
    cases = [
        ("disc", catalog("disc"), identity_tensor(2), [0.4, 0.3], 1e-7),
        ("annulus", catalog("annulus"), identity_tensor(2), [0.9, 0.0], 1e-9),
        ("five", catalog("disc_five_holes"), identity_tensor(2), [0.8, 0.2], 1e-8),
        ("square_hole", catalog("square_hole"), identity_tensor(2), [-0.4, 0.6], 1e-7),
        ("square_hole_aniso", catalog("square_hole"), make_tensor(ANISO_K), [-0.4, 0.6], 1e-7),
        ("shell3d", catalog("shell3d"), identity_tensor(3), [0.8, 0.1, 0.0], 1e-8),
    ]
    data = {"names": np.array([c[0] for c in cases])}
    for name, dom, kt, pole, eps in cases:
        g = backend.pack_geometry(dom)
        ks = np.ascontiguousarray(kt.k_sqrt)
        pole = np.asarray(pole, dtype=float)
        x, st, comp, err = impl.walk_exits_chunk(g.gi, g.gf, g.comp_side, ks, pole, 2, 10, 210,
                                                 99, eps, 10**6)
        assert err == -1
        side0, side1 = _sides(backend, dom, eps)
        o0 = np.zeros(side0.size)
        o1 = np.zeros(side1.size)
        stats = impl.accumulate_chunk(g.gi, g.gf, g.comp_side, ks, pole, 0, 0, 3000, 7, eps,
                                      10**6, side0.anchors, side0.blk, side0.blkf, 0,
                                      side0.idw_radii, 2, side1.anchors, side1.blk,
                                      side1.blkf, 0, side1.idw_radii, 2, o0, o1)
        pre = name + "."
        data.update({pre + "gi": g.gi, pre + "gf": g.gf, pre + "comp_side": g.comp_side,
                     pre + "ksqrt": ks, pre + "pole": pole, pre + "eps": np.float64(eps),
                     pre + "x": x, pre + "steps": st, pre + "comp": comp,
                     pre + "a0": side0.anchors, pre + "blk0": side0.blk, pre + "blkf0": side0.blkf,
                     pre + "a1": side1.anchors, pre + "blk1": side1.blk, pre + "blkf1": side1.blkf,
                     pre + "out0": o0, pre + "out1": o1,
                     pre + "stats": np.array(stats, dtype=np.int64)})
    # budget error: annulus, max_steps = 2 (T/test_backend.py:184-198)
    dom = catalog("annulus")
    g = backend.pack_geometry(dom)
    side0, side1 = _sides(backend, dom, 1e-10)
    res = impl.accumulate_chunk(g.gi, g.gf, g.comp_side, np.eye(2), np.array([0.95, 0.0]), 0,
                                0, 50, 1, 1e-10, 2, side0.anchors, side0.blk, side0.blkf, 0,
                                side0.idw_radii, 2, side1.anchors, side1.blk, side1.blkf, 0,
                                side1.idw_radii, 2, np.zeros(side0.size), np.zeros(side1.size))
    data["budget_err"] = np.int64(res[4])
    np.savez_compressed(OUT / "cases.npz", **data)

    # ---- IDW weight families (T/test_backend.py:132-140 cases; S/_kernel.pyx:323-369) ----
    from exitmeasure.geometry import side_points as _sp
    from exitmeasure.weights import idw_radii_for

    idw = {}
    for name, dom, kt, pole, eps in (cases[1], cases[3]):
        d = dom.dimension
        a1 = _sp(dom, "gamma1", [60] * len(dom.gamma1))
        s1 = backend.pack_side(a1, d, eps, "idw", idw_radii_for(a1), 2)
        a0 = _sp(dom, "gamma0", [80 * len(dom.gamma0)])
        s0 = backend.pack_side(a0, d, eps, "idw", idw_radii_for(a0), 3)
        g = backend.pack_geometry(dom)
        ks = np.ascontiguousarray(kt.k_sqrt)
        pole = np.asarray(pole, dtype=float)
        # chunk contract: in place from non-zero initial values
        o0 = np.linspace(0.0, 1.0, s0.size)
        o1 = np.linspace(0.5, 2.0, s1.size)
        init0, init1 = o0.copy(), o1.copy()
        st = impl.accumulate_chunk(g.gi, g.gf, g.comp_side, ks, pole, 0, 0, 3000, 7, eps, 10**6,
                                   s0.anchors, s0.blk, s0.blkf, 1, s0.idw_radii, s0.idw_power,
                                   s1.anchors, s1.blk, s1.blkf, 1, s1.idw_radii, s1.idw_power,
                                   o0, o1)
        # driver: two poles x 10000 walks (two 8192-chunks per pole)
        poles2 = np.stack([pole, pole * 0.9])
        r = backend.run_accumulate(dom, ks, poles2, 11, eps, 10**6, 10000, s0, s1, threads=4)
        pre = "idw_" + name + "."
        idw.update({pre + "gi": g.gi, pre + "gf": g.gf, pre + "comp_side": g.comp_side,
                    pre + "ksqrt": ks, pre + "pole": pole, pre + "eps": np.float64(eps),
                    pre + "a0": s0.anchors, pre + "blk0": s0.blk, pre + "blkf0": s0.blkf,
                    pre + "r0": s0.idw_radii, pre + "a1": s1.anchors, pre + "blk1": s1.blk,
                    pre + "blkf1": s1.blkf, pre + "r1": s1.idw_radii,
                    pre + "init0": init0, pre + "init1": init1, pre + "out0": o0,
                    pre + "out1": o1, pre + "stats": np.array(st, dtype=np.int64),
                    pre + "poles2": poles2, pre + "raw0": r.raw0, pre + "raw1": r.raw1,
                    pre + "rsteps": r.steps_sum, pre + "rfb": np.int64(r.idw_fallbacks)})
    np.savez_compressed(OUT / "idw.npz", **idw)

    # ---- BASELINE configs in the reference expression (reduced size) ----
    sys.path.insert(0, str(ROOT))
    from paper_2409_03686_b200 import configs

    plan = {1: (32, 2000), 2: (64, 200), 3: (64, 100), 4: (32, 40)}
    out = {}
    for idx, (n_poles, n_rep) in plan.items():
        cfg = configs.get(idx).subset(n_poles, n_rep)
        kt = make_tensor(cfg.kt.k if not cfg.kt.is_identity else np.eye(cfg.d))
        if idx == 3:
            dom = catalog("annulus")
            from exitmeasure.geometry import side_points

            s0 = backend.pack_side(side_points(dom, "gamma0", [512]), 2, cfg.eps)
            s1 = backend.pack_side(side_points(dom, "gamma1", [512]), 2, cfg.eps)
        else:
            outer = (Ball(np.zeros(cfg.d), 1.0) if idx in (1, 4)
                     else Box(np.array([0.5, 0.5]), 0.5))
            dom = make_domain(outer, gamma0=())
            pts = np.ascontiguousarray(cfg.fam1.points)
            generic = BoundaryPointSet(pts, np.zeros(len(pts), dtype=int),
                                       np.arange(len(pts), dtype=float), ())
            s0 = backend.pack_side(None, cfg.d, cfg.eps)
            s1 = backend.pack_side(generic, cfg.d, cfg.eps)
        r = backend.run_accumulate(dom, kt.k_sqrt, cfg.poles, cfg.seed, cfg.eps, 10**6, n_rep,
                                   s0, s1, threads=os.cpu_count())
        pre = f"cfg{idx}."
        out.update({pre + "poles": cfg.poles, pre + "ksqrt": np.ascontiguousarray(kt.k_sqrt),
                    pre + "seed": np.uint64(cfg.seed), pre + "n_rep": np.int64(n_rep),
                    pre + "eps": np.float64(cfg.eps),
                    pre + "raw0": r.raw0.astype(np.int32), pre + "raw1": r.raw1.astype(np.int32),
                    pre + "steps_sum": r.steps_sum, pre + "steps_sq": r.steps_sq_sum,
                    pre + "steps_max": r.steps_max, pre + "anchors1": s1.anchors})
        print(f"cfg{idx}: {n_poles} poles x {n_rep} walks, mean steps "
              f"{r.steps_sum.sum() / (n_poles * n_rep):.2f}")
    np.savez_compressed(OUT / "baseline_cfg.npz", **out)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
