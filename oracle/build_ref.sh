#!/usr/bin/env bash
# Builds the UNMODIFIED reference package (exitmeasure 0.1.0, /root/reference/pkg)
# into oracle/_ref/ so tests, smoke() and bench.py --impl reference can time and
# check against the reference's own compiled Cython kernel.
#
# - Sources are read where they lie; the build runs on a scratch copy under /tmp
#   because setuptools writes build artefacts into the source tree, and
#   /root/reference is read-only.
# - Output goes only to oracle/_ref/ (git-ignored; it still travels to the GPU
#   box with the gpurun snapshot).
# - CFLAGS pin -O2 -ffp-contract=off so the reference's FP64 arithmetic is not
#   FMA-contracted (the SURVEY's F1 bit-reproducibility condition).
# - This is test infrastructure: nothing on the product path imports it.
# - The reference's own test suite is copied beside it (oracle/_ref/ref_tests,
#   same git-ignore / travel rules) so tests/test_gpu_refsuite.py can run it
#   on the GPU box against this backend (the box has no /root/reference).
#   `build_ref.sh --tests-only` refreshes just that copy.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REFERENCE_ROOT:-/root/reference}/pkg"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF absent (GPU box?) - keeping prebuilt $OUT" >&2
  exit 0
fi
copy_tests() {
  rm -rf "$OUT/ref_tests"
  cp -r "$REF/tests" "$OUT/ref_tests"
  # the reference's pytest settings (R/pkg/pyproject.toml [tool.pytest.ini_options])
  printf '[pytest]\naddopts = -m "not nightly"\nmarkers =\n    nightly: long-running checks\n    slow: heavier statistical tests\n' > "$OUT/ref_tests/pytest.ini"
}
if [ "${1:-}" = "--tests-only" ]; then
  copy_tests
  exit 0
fi
TMP="$(mktemp -d /tmp/emref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
rm -rf "$OUT"
mkdir -p "$OUT"
CFLAGS="-O2 -ffp-contract=off" python -m pip install --quiet --no-index \
  --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$OUT" "$TMP/pkg"
copy_tests
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import exitmeasure.backend as b
assert b.BACKEND == "compiled", b.BACKEND
print("oracle/_ref: exitmeasure", b.BACKEND, "kernel at", b._impl.__file__)
PY
