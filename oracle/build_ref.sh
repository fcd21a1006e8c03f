#!/usr/bin/env bash
# Build the reference's own compiled conv kernel into oracle/_ref/ —
# TEST INFRASTRUCTURE ONLY (CPU baseline "kind": "reference").
#
# Source: /root/reference/pkg/src/voxplan/_kernels.pyx + convcore.h, compiled
# where they lie (read-only, nothing is copied into the repo).  The module is
# self-contained (imports nothing from voxplan), so it is loaded standalone by
# oracle/ref_engine.py.  The reference's own build (pkg/setup.py:36-43) uses
# -O3 -march=native; this recipe uses -O3 -march=x86-64-v3 (AVX2 + FMA, the
# width convcore.h's 8-lane vectors need) so the .so also runs on the GPU
# box's host CPU.  Outputs go to oracle/_ref/ only (git-ignored, but shipped
# to the GPU box by gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF_SRC:-/root/reference/pkg/src/voxplan}"
OUT="$HERE/_ref"
PY="${PYTHON:-python}"
if [ ! -f "$REF/_kernels.pyx" ]; then
  echo "reference sources not found at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT"
SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
"$PY" -m cython -3 -o "$OUT/_kernels.c" "$REF/_kernels.pyx"
gcc -O3 -march=x86-64-v3 -fPIC -shared -I"$REF" -I"$PYINC" \
    "$OUT/_kernels.c" -o "$OUT/_kernels$SUFFIX" -lm
echo "$OUT/_kernels$SUFFIX"
