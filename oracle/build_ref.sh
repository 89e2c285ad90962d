#!/usr/bin/env bash
# Build the UNMODIFIED reference package (mtbalign 0.1.0, Python + one Cython
# kernel file) from /root/reference/pkg into oracle/_ref/ with its own setup.py
# flags (-O3).  Test/bench infrastructure only: oracle/_ref is git-ignored but
# travels to the GPU box with the gpurun snapshot, where bench.py --impl
# reference and the cpu_baseline leg import it.  Nothing here is product code.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${MTB_REFERENCE_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference sources not present at $SRC; keeping prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/mtbref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"          # /root/reference is read-only; build from a scratch copy
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$OUT" "$TMP/pkg"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import mtbalign
from mtbalign import kernels
assert kernels.native_available(), "reference Cython engine did not build"
print("oracle/_ref: mtbalign", mtbalign.__version__, "engine", kernels.engine_name())
PY
