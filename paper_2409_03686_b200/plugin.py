"""Install this backend into the reference package, without editing it.

The reference selects its kernel once at import (S/backend.py:24-41, S/ =
/root/reference/pkg/src/exitmeasure/) but resolves every call through module
attributes at call time: ``mc_rem`` calls ``backend.run_accumulate``
(S/estimator.py:21,149), ``batch_exits`` calls ``backend.run_exits``
(S/walk.py:21,123), the driver calls ``_impl.accumulate_chunk`` /
``_impl.walk_exits_chunk`` (S/backend.py:162,213), and the CLI records
``backend.BACKEND`` (S/cli.py:479).  ``install()`` swaps those attributes, so
the reference's CLI, ``mc_rem`` and tests run unchanged on the GPU.

``linalg="device"`` also moves the large dense algebra to the GPU (SURVEY
§8f item 3): ``estimator._gram`` (S/estimator.py:112-118), the SVD of the
scaled operator (``tsvd.svd``, ``linalg.svd``: S/tsvd.py:104,143,
S/cli.py:368) and the Gram eigendecomposition (``tsvd.sym_eig``,
S/tsvd.py:55,158).  The 3x3 ``sym_eig`` behind K^{1/2} stays on the host.

Precision: the default ``"ref64"`` keeps the reference's results bit for bit
(same counts, exits, step statistics and CSVs); ``precision="fp32"`` selects
the production kernel (statistically identical A, much faster).  Subprocess
entry: ``python -m paper_2409_03686_b200.plugin <exitmeasure CLI args>``.
"""

from __future__ import annotations

import sys
import types

import numpy as np

from . import backend as B
from .errors import WalkBudgetError


def _reference_errors():
    try:
        from exitmeasure import errors

        return errors.WalkBudgetError
    except Exception:  # pragma: no cover - reference absent
        return WalkBudgetError


def install_linalg(device: int | None = None):
    """Route the reference's Gram / SVD / Gram-eigendecomposition through
    spectral.py on the GPU (float64; agrees with the host to rounding)."""
    from exitmeasure import estimator, linalg, tsvd

    from . import spectral

    def _gram(a1, sigma1, nu):
        return spectral.gram(a1, sigma1, nu, device)

    def svd(b):
        linalg._require_matrix(b, "B")  # the reference's own checks and errors
        return spectral.svd(b, device)

    def sym_eig(a):
        a = linalg._require_matrix(a, "A")
        n, m = a.shape
        if n != m:
            raise linalg.ValidationError(f"A must be square, got {n}x{m}")
        scale = np.max(np.abs(a)) or 1.0
        if np.max(np.abs(a - a.T)) > 1e-12 * scale:
            raise linalg.ValidationError("A is not symmetric to 1e-12 relative")
        w, v = spectral.sym_eig(a, device)
        return linalg.SymEig(w, v)

    estimator._gram = _gram
    tsvd.svd = svd
    tsvd.sym_eig = sym_eig
    linalg.svd = svd


def install(precision: str | None = None, chain: str | None = None, device: int | None = None,
            module=None, linalg: str | None = None, cache: bool = True):
    """Patch ``exitmeasure.backend`` (or ``module``) to run on this library
    (and, with ``linalg="device"``, the dense algebra: install_linalg).
    ``cache=False`` builds and uploads a fresh plan on every call (no
    resident-plan reuse across calls).  Returns the patched backend module."""
    if linalg not in (None, "host", "device"):
        raise ValueError(f"linalg must be 'host' or 'device', got {linalg!r}")
    if linalg == "device":
        install_linalg(device)
    if module is None:
        import exitmeasure.backend as module
    ref_budget = _reference_errors()

    def run_accumulate(dom, ksqrt, poles, seed, eps, max_steps, n_rep, side0, side1,
                       threads=None):
        try:
            res = B.run_accumulate(dom, ksqrt, poles, seed, eps, max_steps, n_rep, side0, side1,
                                   threads, precision=precision, chain=chain, device=device,
                                   cache=cache, rows="float64")
        except WalkBudgetError as e:
            raise ref_budget(e.pole, e.replicate, e.max_steps) from None
        return module.AccumulateResult(res.raw0, res.raw1, res.steps_sum, res.steps_sq_sum,
                                       res.steps_max, res.idw_fallbacks)

    def run_exits(dom, ksqrt, pole_xy, pole_index, seed, eps, max_steps, n_rep, threads=None):
        try:
            return B.run_exits(dom, ksqrt, pole_xy, pole_index, seed, eps, max_steps, n_rep,
                               threads, precision=precision, chain=chain, device=device)
        except WalkBudgetError as e:
            raise ref_budget(e.pole, e.replicate, e.max_steps) from None

    impl = types.ModuleType("exitmeasure_b200_impl")
    impl.walk_exits_chunk = B.walk_exits_chunk
    impl.accumulate_chunk = B.accumulate_chunk
    if not hasattr(module, "_em_b200_original"):  # keep the reference's own entry points
        module._em_b200_original = {k: getattr(module, k) for k in
                                    ("run_accumulate", "run_exits", "_impl", "BACKEND")}
    module.run_accumulate = run_accumulate
    module.run_exits = run_exits
    module._impl = impl
    module.BACKEND = "cuda-" + (precision or B.default_precision())
    return module


def uninstall(module=None):
    """Restore the reference's own backend entry points (after install)."""
    if module is None:
        import exitmeasure.backend as module
    orig = getattr(module, "_em_b200_original", None)
    if orig:
        for k, v in orig.items():
            setattr(module, k, v)
        del module._em_b200_original
    return module


def main(argv=None):
    """Run the reference CLI with this backend installed."""
    install()
    from exitmeasure import cli

    return cli.main(argv if argv is not None else sys.argv[1:])


if __name__ == "__main__":
    sys.exit(main())
