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
# tests/data/golden.gaes is absent from the mount; regenerate
# it with the reference's own compiled backend and keep it only if it has
# the SHA-256 pinned at test_container.py:26.
mkdir -p "$REPO/baseline/_ref_tests/data"
( cd "$REPO/baseline/_ref_tests" && PYTHONDONTWRITEBYTECODE=1 PYTHONPATH="$REPO/baseline/_ref:." python - <<'PY'
import hashlib
from test_container import GOLDEN, GOLDEN_SHA256, build_golden
blob = build_golden()
if hashlib.sha256(blob).hexdigest() == GOLDEN_SHA256:
    GOLDEN.write_bytes(blob)
    print("golden.gaes regenerated, sha256 matches the pinned digest")
else:
    print("golden.gaes NOT written: digest mismatch")
PY
)
echo "staged: $(ls "$REPO/baseline/_ref/gaes" | wc -l) package files, $(ls "$REPO/baseline/_ref_tests" | wc -l) test files"
