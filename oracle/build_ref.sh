#!/usr/bin/env bash
# Builds the UNMODIFIED reference package (arXiv 1509.06957 MRPT, /root/reference/pkg)
# into oracle/_ref/ so tests, smoke() and bench.py's reference/cpu_baseline legs can
# import it as `mrpt` (compiled Cython backend, -O3 -ffp-contract=off per
# pkg/setup.py:37-39).  The reference tree is read-only, so the build runs from a
# scratch copy under /tmp; only the installed package lands in oracle/_ref/
# (git-ignored, NOT gpurun-ignored, so it travels to the GPU box).
# No reference source is copied into the repository history.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${MRPT_REFERENCE_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC not present; keeping prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/mrpt_ref_build.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$OUT" "$TMP/pkg" >&2
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import mrpt
from mrpt import _kernels
assert _kernels.backend() == "compiled", "reference compiled backend missing"
print("build_ref: mrpt", mrpt.__version__, "backend", _kernels.backend(), file=sys.stderr)
PY
