"""Runs the REFERENCE's own test suite on this backend (tests/test_gpu_refsuite.py).

Put this directory first on PYTHONPATH with EM_B200_REFSUITE=1: every Python
process started under it -- pytest and the ``python -m exitmeasure.cli``
subprocesses the reference's tests spawn (T/test_backend.py:177-195,
T/test_acceptance.py:310-330) -- then resolves the reference's compiled
kernel module ``exitmeasure._kernel`` (the ``_impl`` chunk contract,
S/_kernel.pyx:376-464) to this library's bit-exact REF64 chunk entry points,
and ``plugin.install(precision="ref64")`` swaps the batched drivers
(S/backend.py:147-227).  EXITMEASURE_BACKEND=fallback keeps the reference's
numpy mirror untouched, so the reference's own "compiled vs fallback"
comparisons become "this GPU backend vs the reference's numpy mirror".
Each patched process appends one line to $EM_B200_REFSUITE_LOG.
Test infrastructure only; nothing on the product path imports it.
"""

import importlib.abc
import importlib.util
import os
import sys
import types

if os.environ.get("EM_B200_REFSUITE") == "1" and \
        os.environ.get("EXITMEASURE_BACKEND", "").lower() not in ("fallback", "python"):
    _root = os.environ["EM_B200_ROOT"]
    if _root not in sys.path:
        sys.path.insert(1, _root)

    class _KernelFinder(importlib.abc.MetaPathFinder, importlib.abc.Loader):
        """exitmeasure._kernel -> this library's REF64 chunk functions."""

        def find_spec(self, name, path, target=None):
            if name == "exitmeasure._kernel":
                return importlib.util.spec_from_loader(name, self)
            return None

        def create_module(self, spec):
            return None

        def exec_module(self, module):
            from paper_2409_03686_b200 import backend as B

            module.walk_exits_chunk = B.walk_exits_chunk
            module.accumulate_chunk = B.accumulate_chunk
            module.__em_b200__ = True

    sys.meta_path.insert(0, _KernelFinder())
    import exitmeasure.backend as _rb  # noqa: E402  (selects _impl = our _kernel)

    from paper_2409_03686_b200 import plugin as _plugin  # noqa: E402

    _plugin.install(precision="ref64", module=_rb)
    _log = os.environ.get("EM_B200_REFSUITE_LOG")
    if _log:
        with open(_log, "a") as f:
            f.write(f"{os.getpid()} {' '.join(sys.argv[:3])} backend={_rb.BACKEND} "
                    f"kernel={getattr(sys.modules['exitmeasure._kernel'], '__em_b200__', False)}\n")
    del types


def _chain_next_sitecustomize():
    """Run the next sitecustomize on sys.path too (this one shadows it), so a
    launcher's own hook (e.g. one that records loaded libraries) still runs."""
    import importlib.util
    from pathlib import Path

    here = Path(__file__).resolve().parent
    for entry in sys.path:
        try:
            cand = Path(entry or ".").resolve() / "sitecustomize.py"
        except OSError:
            continue
        if cand.parent == here or not cand.is_file():
            continue
        spec = importlib.util.spec_from_file_location("_em_chained_sitecustomize", cand)
        mod = importlib.util.module_from_spec(spec)
        try:
            spec.loader.exec_module(mod)
        except Exception:  # a foreign hook's failure must not break the suite
            pass
        return


_chain_next_sitecustomize()
