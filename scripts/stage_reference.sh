#!/usr/bin/env bash
# Stage the reference package for the drop-in tests (run here, where
# /root/reference is mounted; the results are git-ignored but ship to the
# GPU box with the gpurun snapshot):
#   baseline/_ref/        pip-installed reference `gaes` (compiled backend)
#   baseline/_ref_tests/  the reference's own test files, run unchanged on
#                         the GPU with `-p paper_1506_08503_b200.plugin`
set -euo pipefail
REPO="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC; nothing to stage"; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg" >/dev/null
rm -rf "$REPO/baseline/_ref_tests"
cp -r "$SRC/tests" "$REPO/baseline/_ref_tests"
rm -rf "$TMP"
echo "staged: $(ls "$REPO/baseline/_ref/gaes" | wc -l) package files, $(ls "$REPO/baseline/_ref_tests" | wc -l) test files"
