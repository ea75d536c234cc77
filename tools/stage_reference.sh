#!/bin/bash
# Stage the UNMODIFIED reference package into baseline/_ref (git-ignored;
# travels to the GPU box with the gpurun snapshot):
#   * the package itself, built with its compiled backend, by the one
#     offline install the task allows (numpy is already in the image, so
#     --no-deps: only dependency resolution fails without it);
#   * the reference's own test suite (pkg/tests) as baseline/_ref/tests, so
#     tools/refsuite/run.py can run it against the B200 implementation.
# The install builds in a copy under /tmp (/root/reference is read-only).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no /root/reference: nothing to stage"; exit 0; }
TMP=$(mktemp -d /tmp/sfdt_ref_stage.XXXXXX)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
touch "$ROOT/baseline/_ref/tests/__init__.py"   # resolve `tests.conftest` to the staged suite
rm -rf "$TMP"
cd /tmp && PYTHONPATH="$ROOT/baseline/_ref" python -c "import sfft_dt; print('staged sfft_dt', sfft_dt.__version__, sfft_dt.BACKEND)"
