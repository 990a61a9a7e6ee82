"""The drop-in: the UNMODIFIED reference package (oracle/_ref) with this
backend installed produces the reference's own results bit for bit -- mc_rem
bundles and the CLI's CSV outputs (the T/test_backend.py:177-195 criterion,
here compiled-CPU vs CUDA instead of compiled vs fallback).  B200 only."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "exitmeasure").exists():
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, str(REF))
    import exitmeasure.backend as rb

    return rb


def _annulus_bundle(n=4000, seed=17):
    from exitmeasure.conductivity import identity_tensor
    from exitmeasure.estimator import make_measurements, mc_rem
    from exitmeasure.geometry import catalog, circle_points, side_points
    from exitmeasure.walk import WalkConfig
    from exitmeasure.weights import voronoi_family

    dom = catalog("annulus")
    fam1 = voronoi_family(side_points(dom, "gamma1", [40]), dom)
    fam0 = voronoi_family(side_points(dom, "gamma0", [80]), dom)
    poles = circle_points(np.zeros(2), 0.95, 8).points
    meas = make_measurements(dom, poles, np.zeros(8))
    return mc_rem(dom, identity_tensor(2), meas, fam1, fam0, WalkConfig(eps=1e-8, seed=seed), n)


def test_mc_rem_bit_identical_through_plugin(ref):
    from paper_2409_03686_b200 import plugin

    saved = (ref.run_accumulate, ref.run_exits, ref._impl, ref.BACKEND)
    cpu = _annulus_bundle()
    try:
        plugin.install(precision="ref64", module=ref)
        assert ref.BACKEND == "cuda-ref64"
        gpu = _annulus_bundle()
    finally:
        ref.run_accumulate, ref.run_exits, ref._impl, ref.BACKEND = saved
    for name in ("a0", "a1", "lambda_nu", "steps_mean", "steps_std", "steps_max"):
        assert np.array_equal(getattr(cpu, name), getattr(gpu, name)), name


def test_budget_error_is_the_reference_class(ref):
    from exitmeasure.errors import WalkBudgetError
    from exitmeasure.geometry import catalog
    from exitmeasure.walk import WalkConfig, batch_exits
    from exitmeasure.conductivity import identity_tensor

    from paper_2409_03686_b200 import plugin

    saved = (ref.run_accumulate, ref.run_exits, ref._impl, ref.BACKEND)
    try:
        plugin.install(precision="ref64", module=ref)
        with pytest.raises(WalkBudgetError):
            batch_exits(catalog("annulus"), identity_tensor(2), [0.95, 0.0],
                        WalkConfig(eps=1e-10, seed=1, max_steps=1), 64)
    finally:
        ref.run_accumulate, ref.run_exits, ref._impl, ref.BACKEND = saved


def test_cli_outputs_byte_identical(ref, tmp_path):
    outs = []
    env = dict(os.environ, PYTHONPATH=f"{REF}:{ROOT}")
    for label, mod in (("cpu", "exitmeasure.cli"), ("gpu", "paper_2409_03686_b200.plugin")):
        out = tmp_path / label
        cmd = [sys.executable, "-m", mod, "--example", "ex5_2", "--solution", "sol2d_2",
               "--n", "2000", "--seed", "9", "--r", "1:3", "--out", str(out)]
        proc = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
        assert proc.returncode == 0, proc.stderr[-3000:]
        outs.append(out)
    for name in ("eigenvalues.csv", "density.csv", "eigvecs.csv", "tsvd.csv", "residuals.csv"):
        assert (outs[0] / name).read_bytes() == (outs[1] / name).read_bytes(), name


def test_reference_driver_threads_over_the_chunk_dropin(ref):
    """Only ``_impl`` swapped: the reference's OWN driver (S/backend.py:147-199,
    a ThreadPoolExecutor over 8192-walk chunks, 8 threads) calls our
    accumulate_chunk / walk_exits_chunk concurrently; results equal the
    reference kernel's bit for bit (reentrancy, released GIL, in-place +=)."""
    from exitmeasure.conductivity import identity_tensor
    from exitmeasure.geometry import catalog, side_points

    from paper_2409_03686_b200 import plugin

    dom = catalog("annulus")
    s0 = ref.pack_side(side_points(dom, "gamma0", [64]), 2, 1e-6)
    s1 = ref.pack_side(side_points(dom, "gamma1", [32]), 2, 1e-6)
    poles = np.array([[0.0, 0.75], [0.8, 0.1], [-0.6, -0.5]])
    args = (dom, identity_tensor(2).k_sqrt, poles, 23, 1e-6, 10**6, 20000, s0, s1)
    cpu = ref.run_accumulate(*args, threads=8)
    x_cpu = ref.run_exits(dom, identity_tensor(2).k_sqrt, poles[1], 1, 23, 1e-6, 10**6, 20000,
                          threads=8)
    saved = (ref.run_accumulate, ref.run_exits, ref._impl, ref.BACKEND)
    try:
        plugin.install(precision="ref64", module=ref)
        ref.run_accumulate, ref.run_exits = saved[0], saved[1]  # keep the reference driver
        assert ref._impl.accumulate_chunk.__module__.startswith("paper_2409_03686_b200")
        gpu = ref.run_accumulate(*args, threads=8)
        x_gpu = ref.run_exits(dom, identity_tensor(2).k_sqrt, poles[1], 1, 23, 1e-6, 10**6, 20000,
                              threads=8)
    finally:
        ref.run_accumulate, ref.run_exits, ref._impl, ref.BACKEND = saved
    for name in ("raw0", "raw1", "steps_sum", "steps_sq_sum", "steps_max"):
        assert np.array_equal(getattr(cpu, name), getattr(gpu, name)), name
    for a, b in zip(x_cpu, x_gpu):
        assert np.array_equal(a, b)


@pytest.mark.slow
def test_five_disc_anchor_through_the_cli(ref, tmp_path):
    """The paper's published accuracy anchor (R/PAPER.md:202-203; acceptance
    C03, T/test_acceptance.py:135-152): the averaged inaccessible exit mass of
    the five-disc geometry ex5_4 over its 100 poles at 1e5 walks per pole,
    read back from the reference CLI's summary.json.  The reference itself
    (compiled Cython kernel) gives 0.1125; REF64 through plugin.install()
    must reproduce its value EXACTLY, FP32 within 4 standard errors of the
    difference of two independent estimates."""
    import json

    from exitmeasure.cli import RunConfig, run

    from paper_2409_03686_b200 import plugin

    def avg(label, eps=None):
        out = tmp_path / label
        run(RunConfig(example="ex5_4", solution="sol2d_3", n=10**5, seed=314, r="1:6",
                      out=str(out), eps=eps))
        s = json.loads((out / "summary.json").read_text())["replicates"][0]
        return float(s["mu_gamma1_avg"])

    mu_ref = avg("reference")
    assert round(mu_ref, 4) == 0.1125
    out = {}
    # ex5_4 runs at eps = 1e-10, below the FP32 kernel's resolution (it
    # refuses such shells); the FP32 arm runs eps = 1e-6, whose eps-shell
    # shift of the exit law (order eps) is ~1e-2 standard errors here
    for prec, eps in (("ref64", None), ("fp32", 1e-6)):
        try:
            plugin.install(precision=prec, module=ref)
            out[prec] = avg(prec, eps)
        finally:
            plugin.uninstall(ref)
    assert out["ref64"] == mu_ref
    # SE of a 100-pole average of binomial fractions near 0.11 at 1e5 walks
    se = np.sqrt(mu_ref * (1 - mu_ref) / 10**5 / 100)
    assert abs(out["fp32"] - mu_ref) <= 4 * np.sqrt(2) * se, (out, mu_ref, se)
