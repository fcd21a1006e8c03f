#!/usr/bin/env bash
# Build the reference engine into oracle/_ref/ — TEST INFRASTRUCTURE ONLY
# (the CPU baseline "kind": "reference" and the reference-side binding tests).
#
# Two artefacts, both from the reference's own, unmodified sources:
#  1. oracle/_ref/voxplan/ — the whole reference package (voxplan: prototxt,
#     PZNW, compiler, PlanRunner, run_tiled, compiled _kernels), installed the
#     standard way (pip install --no-deps --no-build-isolation --target) from a
#     scratch copy of /root/reference/pkg (its build writes into the source
#     tree, and /root/reference is read-only).  BASELINE.md §2's CPU arm is
#     voxplan.PlanRunner(plan, backend="compiled") / run_tiled from here.
#  2. oracle/_ref/_kernels*.so — the reference's _kernels.pyx + convcore.h
#     alone (self-contained, loaded standalone by oracle/ref_engine.py).
# The reference's build (pkg/setup.py:36-43) uses -O3 -march=native; the GPU
# box's host CPU may lack this container's ISA extensions, so both kernel
# modules are (re)built with -O3 -march=x86-64-v3 (AVX2 + FMA: the width
# convcore.h's 8-lane vectors need).  Outputs go to oracle/_ref/ only
# (git-ignored, shipped to the GPU box by gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
PKG="${REF_PKG:-/root/reference/pkg}"
REF="$PKG/src/voxplan"
OUT="$HERE/_ref"
PY="${PYTHON:-python}"
if [ ! -f "$REF/_kernels.pyx" ]; then
  echo "reference sources not found at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT"
SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"

build_kernels() {   # $1 = output .so
  local tmpc
  tmpc="$(mktemp -d)"
  "$PY" -m cython -3 -o "$tmpc/_kernels.c" "$REF/_kernels.pyx"
  gcc -O3 -march=x86-64-v3 -fPIC -shared -I"$REF" -I"$PYINC" -I"$($PY -c 'import numpy; print(numpy.get_include())')" \
      "$tmpc/_kernels.c" -o "$1" -lm
  rm -rf "$tmpc"
}

# 2. standalone kernel module
build_kernels "$OUT/_kernels$SUFFIX"

# 1. the whole package
SCRATCH="$(mktemp -d)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$PKG" "$SCRATCH/pkg"
rm -rf "$OUT/voxplan" "$OUT"/voxplan-*.dist-info "$OUT/bin"
"$PY" -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$OUT" \
    "$SCRATCH/pkg" >&2
rm -f "$OUT/voxplan/_kernels.c"
build_kernels "$OUT/voxplan/_kernels$SUFFIX"
echo "$OUT/_kernels$SUFFIX"
echo "$OUT/voxplan"
