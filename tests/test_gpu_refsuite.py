"""The reference's OWN hot-path test suite, unmodified, on this backend.

oracle/build_ref.sh copies the reference's tests (T/) beside the built
reference (oracle/_ref/ref_tests; git-ignored, travels to the GPU box).
They run here under tests/refsuite/sitecustomize.py, which resolves the
reference's compiled kernel module to this library's bit-exact REF64 chunk
entry points and installs the batched GPU drivers -- in pytest and in every
CLI subprocess the tests spawn.  Suite: T/test_rng.py, T/test_backend.py
(compiled-vs-fallback bit identity: now GPU vs the reference's numpy mirror;
pruned vs brute-force binning; chunk-split invariance; budget errors; CLI
byte-identity), T/test_walk.py (scalar replay, analytic oracles,
containment), T/test_estimator.py, and T/test_acceptance.py (C01-C12,
including the five-disc anchor C03 and the worker-count determinism C12).
SURVEY §8b:441 / §7 step 2."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"
SUITE = ["test_rng.py", "test_backend.py", "test_benchmark.py", "test_walk.py", "test_estimator.py",
         "test_acceptance.py"]


@pytest.mark.skipif(not (REF / "ref_tests").exists(), reason="oracle/_ref/ref_tests not built")
def test_reference_suite_passes_on_gpu_backend(tmp_path):
    from paper_2409_03686_b200 import _native

    _native.require_device(0)
    log = tmp_path / "patched.log"
    env = dict(os.environ, EM_B200_REFSUITE="1", EM_B200_ROOT=str(ROOT),
               EM_B200_REFSUITE_LOG=str(log),
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "refsuite"), str(REF), str(ROOT)]
                                          + [p for p in os.environ.get("PYTHONPATH", "").split(
                                              os.pathsep) if p]))
    env.pop("EXITMEASURE_BACKEND", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-s", "-p", "no:cacheprovider", "-rfE"] + SUITE
    res = subprocess.run(cmd, cwd=REF / "ref_tests", env=env, capture_output=True, text=True,
                         timeout=1800)
    out = res.stdout + res.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "refsuite.log").write_text(out + "\n--- patched ---\n" +
                                                      (log.read_text() if log.exists() else ""))
    assert res.returncode == 0, out[-6000:]
    assert " passed" in out and " failed" not in out
    lines = log.read_text().splitlines()
    # pytest itself and the CLI subprocesses ran on the GPU backend
    assert all("backend=cuda-ref64 kernel=True" in l for l in lines), lines
    assert any("--example" in l for l in lines), lines  # python -m exitmeasure.cli ...
