#!/usr/bin/env bash
# Build the UNMODIFIED reference package (certkv, /root/reference/pkg) with its
# Cython kernel backend (_kernels/_core.pyx -> C -> .so) into oracle/_ref/.
#
# TEST / BASELINE INFRASTRUCTURE ONLY: oracle/_ref is the CPU arm of bench.py
# (--impl reference, cpu_baseline kind "reference") and nothing else.  The
# output is git-ignored (never committed) but travels to the GPU box with the
# repo snapshot; /root/reference itself is read-only and absent on the box, so
# the build runs here, from a scratch copy of the sources (setup.py writes the
# generated C next to the .pyx).  No reference source is copied into the repo's
# history.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${CKV_REFERENCE_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
[ -d "$SRC" ] || { echo "reference sources not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/certkv_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT.tmp"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$OUT.tmp" "$TMP/pkg"
rm -rf "$OUT"
mv "$OUT.tmp" "$OUT"
# record what was built
PYTHONPATH="$OUT" python - <<'PY' > "$OUT/BUILD_INFO.txt"
import certkv, certkv._kernels as k
print("certkv", getattr(certkv, "__version__", "?"), "backend:", k.get_backend().NAME,
      "available:", k.available_backends())
PY
cat "$OUT/BUILD_INFO.txt"
