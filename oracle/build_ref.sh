#!/usr/bin/env bash
# Build the UNMODIFIED reference package (bermuda, with its Cython path walker)
# into oracle/_ref/ so tests and bench.py's reference arm can run the real thing.
# Test infrastructure only: nothing under paper_0805_1827_b200/ imports it.
# The reference source tree is read-only, so the build runs from a /tmp copy.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC not present; keeping prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/bermuda_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$OUT" "$TMP/pkg"
PYTHONPATH="$OUT" python -c "import bermuda; from bermuda._kernels import available_backends as a; assert 'cython' in a(), a(); print('oracle/_ref: bermuda', bermuda.__version__, a())"
