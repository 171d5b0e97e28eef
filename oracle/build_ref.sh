#!/usr/bin/env bash
# Build the reference's own native hot-path kernel into oracle/_ref/.
#
# TEST INFRASTRUCTURE ONLY.  The reference's single native component is
# pkg/src/gaes/_kernel.pyx (Cython -> C, compiled with -O3 by
# pkg/setup.py:42-51).  We compile it from the source where it lies under
# /root/reference -- nothing is copied into the repo -- and write only into
# oracle/_ref/ (git-ignored, shipped to the GPU box with the snapshot).
# The module is self-contained (no imports from the gaes package), so
# `import _kernel` from oracle/_ref gives the reference's cbc_encrypt /
# cbc_decrypt with its exact 7-argument contract.  bench.py --impl reference
# and the cpu_baseline leg time it; tests use it to pin the C oracle.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${GAES_REFERENCE_ROOT:-/root/reference}/pkg/src/gaes/_kernel.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "reference source $SRC not present; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
PY="${PYTHON:-python3}"
mkdir -p "$OUT"
SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
INC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
TARGET="$OUT/_kernel$SUFFIX"
if [ -f "$TARGET" ] && [ "$TARGET" -nt "$SRC" ]; then
  exit 0
fi
"$PY" -m cython -3 "$SRC" -o "$OUT/_kernel.c"
gcc -O3 -fPIC -shared -fwrapv -fno-strict-aliasing -DNDEBUG -I"$INC" \
    "$OUT/_kernel.c" -o "$TARGET"
echo "built $TARGET"
